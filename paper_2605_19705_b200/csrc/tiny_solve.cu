// Whole-solve persistent kernel for the tiny network of BASELINE config C1 (1 x 32 x 32 image,
// N(x) = x + c3(sp(c2(sp(c1(x))))), widths 1 -> 16 -> 16 -> 1, periodic blur, gradient step):
// the i-DEQ loop of Alg. 1 -- extrapolation (Eq. 4), the network and
// its input VJP (Eq. 2), the fidelity gradient A^T(Az - y), the update (Alg. 1 l.8,
// P:219), the residual ||x^{k+1} - x^k|| / ||x^k|| and the stop rule -- runs for all
// iterations inside ONE launch. The per-iteration path costs ~11 launches (72 us per iteration,
// launch- and latency-bound); here every operand stays in shared memory.
//
// One image = one thread-block cluster of P CTAs (a batch runs one cluster per image): P = 16
// (non-portable cluster size, 2 rows per CTA at H = 32) where H allows, else 8. CTA r owns rows
// [r R, (r + 1) R) of the image (R = H / P) and keeps every tensor of the iteration for those rows
// plus halo rows above and below. A stage's producer PUSHES its boundary rows straight into the
// halo rows of the CTAs that read them (st.shared::cluster, DSMEM; the 9x9 blur's 4-row halo reaches
// two CTAs up and down at R = 2) as it computes them, so one cluster barrier per stage both
// publishes a tensor and completes every halo -- no copy phase. Cheap layers are recomputed on the
// halo rows instead of exchanged (a1 and U on rows -1 and R), which removes two of the barriers,
// and the residual's barrier also completes the next iteration's z halos: 5 per iteration. The
// first barrier is split: its arrive follows the pushed A z - y rows, and a1 (local) is computed
// before the wait. The
// residual's three partial sums are pushed into every CTA and summed in fp64 by a fixed butterfly,
// so all P CTAs take the identical stop decision.
//
// Layouts: the network tensors (a1, a2, q2, q1 with 16 channels, U) are planes of (R + 4) rows x
// (W + 2) columns (channel pitch padded to 2 mod 32 words: the 4 lanes of a pixel read 4 channel
// planes in distinct banks) whose border (columns -1 and W, and halo rows outside the image) is
// zero, so the 3x3 convolutions read without bounds checks. The blur operands (z, the residual rb)
// are planes of (R + 2 kc) rows x (W + 2 kc) columns with PERIODIC borders (the blur is a circular
// convolution, reading Q9); c1 reads z through an explicit zero-padding mask. The 16 -> 16
// convolutions give a work item 2 rows x 4 output channels (register blocking: 12 input and 9
// weight loads per 72 FMAs), split over all 512 threads by input channel (4 K parts at R = 2, 2 at
// R = 4) whose partial sums meet in shared memory, every thread finishing 8 / ksplit outputs (the
// blur adjoint A^T rb moved to stage [4], whose q2 items leave threads idle); the single-channel
// outputs and the blur split the contraction over adjacent lanes, combined by fixed-order shuffles. x^k and the candidate x^{k+1} are ping-pong planes.
//
// Measured (B200, C1, tools/tiny_prof.cu): 18.8 us per iteration with 8-CTA clusters -> 12.9 us
// with 16-CTA clusters, conflict-free channel planes, the unrolled 9x9 blur and SFU softplus.
//
// fp32 throughout (the FFMA path's arithmetic; softplus and sigmoid from the SFU exp / log, abs.
// error ~1e-7), matching the fp32 parity mode. Supported: TINY3 with hidden width 16, C = 1,
// identity skip, softplus, direct blur gradient step, per-image stop rule, no restart / averaging
// (the runtime falls back otherwise).
#include "common.cuh"
#include "kernels.h"

namespace ideq {

constexpr int TS_PMAX = 16;  // CTAs per image (cluster size P: 16 where the image allows, else 8)
constexpr int TS_T = 512;    // threads per CTA: 4 per pixel for R x W = 128
constexpr int TS_C = 16;     // hidden width

__device__ __forceinline__ uint32_t ts_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint32_t ts_mapa(uint32_t addr, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(rank));
  return out;
}
__device__ __forceinline__ float ts_ld_cluster(uint32_t a) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void ts_st_cluster(uint32_t a, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory");
}
__device__ __forceinline__ void ts_cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void ts_cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void ts_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t ts_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// Shared-memory layout (floats).
struct TsLayout {
  int R, W, kc;
  int WP, PN;      // network planes: pitch W + 2, (R + 4) rows (2 halo rows each side), padded so
                   // that the 4 lanes of a pixel reading 4 channel planes hit 4 distinct banks
  int WB, PB, HB;  // blur planes: pitch W + 2 kc, (R + 2 HB) rows, HB = max(kc, 1)
  int z, rb, u, a1, a2, q2, q1;
  int xk, gf, xn, y;
  int w1f, w2f, w3f, w1t, w2t, w3t, kern, red, part;
  int total;
  __host__ __device__ void init(int R_, int W_, int ks) {
    R = R_; W = W_; kc = (ks - 1) / 2;
    HB = kc > 1 ? kc : 1;
    WP = W + 2; PN = (R + 4) * WP;
    PN += (2 - PN % 32 + 32) % 32;  // PN = 2 (mod 32): channel planes 4q + j start 8q banks apart
    WB = W + 2 * kc; PB = (R + 2 * HB) * WB;
    int o = 0;
    auto take = [&](int n) { const int b = o; o += (n + 3) & ~3; return b; };
    z = take(PB); rb = take(PB); u = take(PN);
    a1 = take(TS_C * PN); a2 = take(TS_C * PN); q2 = take(TS_C * PN); q1 = take(TS_C * PN);
    xk = take(R * W); gf = take(R * W); xn = take(R * W); y = take(R * W);
    w1f = take(9 * TS_C); w2f = take(TS_C * 9 * TS_C); w3f = take(TS_C * 9);
    w1t = take(TS_C * 9); w2t = take(TS_C * 9 * TS_C); w3t = take(9 * TS_C);
    kern = take(ks * ks); red = take(TS_PMAX * 4); part = take(TS_T * 8);
    total = o;
  }
  __device__ int n_at(int plane, int ch, int r, int c) const { return plane + ch * PN + (r + 2) * WP + c + 1; }
  __device__ int b_at(int plane, int r, int c) const { return plane + (r + HB) * WB + c + kc; }
};

#ifndef TS_PROF
#define TS_PROF 0
#endif
__device__ long long ts_prof[16];  // TS_PROF builds: clock64 per stage, summed over iterations (CTA 0)
#define TS_MARK(i)                                                   \
  if (TS_PROF && blockIdx.x == 0 && threadIdx.x == 0) {              \
    const long long now = clock64();                                 \
    ts_prof[i] += now - t_mark;                                      \
    t_mark = now;                                                    \
  }

struct TinyArgs {
  int N, H, W, R, ks, kper;
  const float* kern;  // [1 or N][ks][ks]
  const float* w1;    // c1 [16][1][3][3]
  const float* w2;    // c2 [16][16][3][3]
  const float* w3;    // c3 [1][16][3][3]
  const float* y;     // [N][H][W]
  float* x;           // in: x^0, out: x-hat
  float lam, tau, beta, tol;
  int max_iter, check_every;
  int* iters;
  float* res;
  int* status;
  float* trace;  // [trace_cap] max_i r_i per iteration (float bits, atomicMax), or null
  int trace_cap;
  int* kdone;    // iterations run by the longest image (atomicMax)
};

// Store v at row r (own, 0 <= r < R), column c of a network plane and push it into the halo rows of
// the CTAs above (their row R + r, if r < nh) and below (their row r - R, if r >= R - nh); image
// borders have no neighbour there (those halo rows stay zero = the convolutions' zero padding).
__device__ __forceinline__ void ts_put_net(float* sm, const TsLayout& L, int o, float v, int r, int rank, int H, int nh,
                                          uint32_t base) {  // nh <= R: the halo rows come from the adjacent CTAs
  sm[o] = v;
  if (r < nh && rank > 0) ts_st_cluster(ts_mapa(base + 4u * (uint32_t)(o + L.R * L.WP), (uint32_t)(rank - 1)), v);
  if (r >= L.R - nh && (rank + 1) * L.R < H)
    ts_st_cluster(ts_mapa(base + 4u * (uint32_t)(o - L.R * L.WP), (uint32_t)(rank + 1)), v);
}
// Store v at (r, c) of a blur plane, its periodic column copies, and push the row into the halo
// rows of every CTA whose halo covers it (periodic in the image: the first CTA's rows are the last
// one's lower halo; with R < HB a row reaches the CTAs d = 1 .. ceil(HB / R) away).
template <int P>
__device__ __forceinline__ void ts_put_blur(float* sm, const TsLayout& L, int plane, int r, int c, float v, int rank,
                                           uint32_t base) {
  int cols[2] = {c, c};
  int nc = 1;
  if (c < L.kc) cols[nc++] = c + L.W;
  else if (c >= L.W - L.kc) cols[nc++] = c - L.W;
  for (int i = 0; i < nc; ++i) {
    sm[L.b_at(plane, r, cols[i])] = v;
    for (int d = 1; (d - 1) * L.R < L.HB && d < P; ++d) {
      const uint32_t up = (uint32_t)((rank + P - d) % P), dn = (uint32_t)((rank + d) % P);
      if (r + d * L.R < L.R + L.HB) ts_st_cluster(ts_mapa(base + 4u * (uint32_t)L.b_at(plane, r + d * L.R, cols[i]), up), v);
      if (r - d * L.R >= -L.HB) ts_st_cluster(ts_mapa(base + 4u * (uint32_t)L.b_at(plane, r - d * L.R, cols[i]), dn), v);
    }
  }
}

// softplus(t) = max(t, 0) + log(1 + e^{-|t|}) and sp'(p) = 1 - e^{-a} from a = sp(p) with the SFU
// exp / log (abs. error ~1e-7: the 1 + u rounding, far below the 1e-4 iterate tolerance of the
// fp32 mode; the accurate log1pf / expm1f sequences cost ~3x the instructions)
__device__ __forceinline__ float ts_softplus(float t) { return fmaxf(t, 0.f) + __logf(1.f + __expf(-fabsf(t))); }
__device__ __forceinline__ float ts_dsp(float a) { return 1.f - __expf(-a); }  // sigmoid(p) from a = sp(p)
// fixed-order sums over the 4 (2) adjacent lanes of one pixel
__device__ __forceinline__ float ts_sum4(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}

// 16 -> 16 3x3 convolution, 2 output rows (r0, r0 + 1) x 4 output channels (4q .. 4q + 3) at column c;
// w: [ci][tap][co] (forward) or, ADJ (conv3x3^T: flipped taps), [co][tap][ci] -- same indexing
// over the input channels [ci0, ci0 + nci)
template <bool ADJ>
__device__ __forceinline__ void ts_conv16(const float* sm, const TsLayout& L, int in_plane, int w, int r0, int c,
                                          int q, int ci0, int nci, float (&acc)[2][4]) {
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[i][e] = 0.f;
#pragma unroll 2
  for (int ci = ci0; ci < ci0 + nci; ++ci) {
    const float* in = sm + L.n_at(in_plane, ci, r0, c);
    float v[4][3];  // input rows r0 - 1 .. r0 + 2, columns c - 1 .. c + 1
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) v[a][b] = in[(a - 1) * L.WP + (b - 1)];
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) {
      const int ta = tap / 3, tb = tap % 3;
      const float x0 = ADJ ? v[2 - ta][2 - tb] : v[ta][tb];
      const float x1 = ADJ ? v[3 - ta][2 - tb] : v[ta + 1][tb];
      const float4 wv = *reinterpret_cast<const float4*>(sm + w + (ci * 9 + tap) * TS_C + 4 * q);
      acc[0][0] = fmaf(wv.x, x0, acc[0][0]); acc[0][1] = fmaf(wv.y, x0, acc[0][1]);
      acc[0][2] = fmaf(wv.z, x0, acc[0][2]); acc[0][3] = fmaf(wv.w, x0, acc[0][3]);
      acc[1][0] = fmaf(wv.x, x1, acc[1][0]); acc[1][1] = fmaf(wv.y, x1, acc[1][1]);
      acc[1][2] = fmaf(wv.z, x1, acc[1][2]); acc[1][3] = fmaf(wv.w, x1, acc[1][3]);
    }
  }
}

// Split-K partials of the blocked 16 -> 16 convolutions: with R = 2 (16-CTA clusters) the blocked
// mapping has only W x 4 items, so ksplit = 2 threads share an item (8 input channels each); the
// second half's 8 accumulators go through shared memory and are added in a fixed order.
// KS: the blur kernel size as a compile-time constant (its loops fully unrolled), 0 = runtime A.ks.
template <int P, int KS>
__global__ void __launch_bounds__(TS_T, 1) tiny_solve_kernel(TinyArgs A) {
  extern __shared__ __align__(16) float sm[];
  const int rank = (int)ts_rank();
  const int n = blockIdx.x / P;
  const int H = A.H, W = A.W, R = A.R;
  const int row0 = rank * R;
  TsLayout L;
  L.init(R, W, A.ks);
  const int RW = R * W;
  const int ks = KS ? KS : A.ks, kc = L.kc;
  const uint32_t base = ts_smem_u32(sm);
  // ---- zero everything (network plane borders stay zero), weights in stage-friendly layouts
  for (int t = threadIdx.x; t < L.total; t += TS_T) sm[t] = 0.f;
  __syncthreads();
  for (int t = threadIdx.x; t < 9 * TS_C; t += TS_T) {
    const int co = t / 9, tap = t % 9;
    sm[L.w1f + tap * TS_C + co] = A.w1[co * 9 + tap];  // c1 [co][0][tap] -> [tap][co]
    sm[L.w1t + co * 9 + tap] = A.w1[co * 9 + tap];     // c1^T: [co][tap]
    sm[L.w3f + co * 9 + tap] = A.w3[co * 9 + tap];     // c3 [0][ci][tap] -> [ci][tap]
    sm[L.w3t + tap * TS_C + co] = A.w3[co * 9 + tap];  // c3^T: [tap][ci]
  }
  for (int t = threadIdx.x; t < TS_C * TS_C * 9; t += TS_T) {
    const int co = t / (TS_C * 9), ci = (t / 9) % TS_C, tap = t % 9;
    sm[L.w2f + (ci * 9 + tap) * TS_C + co] = A.w2[t];  // c2: [ci][tap][co]
    sm[L.w2t + (co * 9 + tap) * TS_C + ci] = A.w2[t];  // c2^T: [co][tap][ci]
  }
  const float* kg = A.kern + (A.kper ? (long long)n * ks * ks : 0);
  for (int t = threadIdx.x; t < ks * ks; t += TS_T) sm[L.kern + t] = kg[t];
  const long long img = (long long)n * H * W + (long long)row0 * W;
  // z^0 = x^0 must be complete in every CTA of the cluster (own rows, pushed halos) before [1]
  ts_cluster_sync();
  for (int t = threadIdx.x; t < RW; t += TS_T) {
    const float v = A.x[img + t];
    sm[L.xk + t] = v;
    sm[L.y + t] = A.y[img + t];
    ts_put_blur<P>(sm, L, L.z, t / W, t % W, v, rank, base);
  }
  int iters = 0, status = 1;
  float res = __int_as_float(0x7fc00000);
  // blocked 16 -> 16 stages: item -> (column, row pair, channel quarter); every thread of the CTA
  // takes part: ksplit = TS_T / nb threads per item (4 at R x W = 64, 2 at 128), each over
  // 16 / ksplit input channels, and each finishes 8 / ksplit of the item's 8 outputs
  const int nb = W * (R / 2) * 4;  // blocked items (R x W <= 128: nb <= TS_T / 2)
  const int ksplit = TS_T / nb;
  const int tb = threadIdx.x % nb, kh = threadIdx.x / nb;  // item, K part
  const int cb = tb % W, rb0 = 2 * ((tb / W) % (R / 2)), qb = tb / (W * (R / 2));
  const int ci0 = kh * (TS_C / ksplit), nci = TS_C / ksplit;
  const int nout = 8 / ksplit;  // outputs i = kh * nout .. (kh + 1) * nout - 1 (row i / 4, channel 4 qb + i % 4)
  // split-K stages: 4 lanes per pixel
  const int pk = threadIdx.x >> 2, qk = threadIdx.x & 3;
  const int rk = pk / W, ck = pk % W;
  const bool act_k = pk < RW;
  int xk_o = L.xk, xn_o = L.xn;  // x^k and the candidate x^{k+1} (ping-pong planes)
  long long t_mark = clock64();
  ts_cluster_sync();  // z^0 (own rows + pushed halos) complete on every CTA
  for (int k = 0; k < A.max_iter; ++k) {
    TS_MARK(0)
    // [1] rb = A z - y (true periodic convolution, reading Q8), pushed to the neighbours' halos, and
    //     the cluster barrier's arrive; then a1 = sp(c1(z)) on rows -1 .. R (the halo rows recomputed
    //     locally; zero outside the image), which needs no neighbour, while the barrier completes
    if (act_k) {  // kernel rows i = qk, qk + 4, ...: (A z)[r][c] = sum k[i][j] z[r - i + kc][c - j + kc]
      float s = 0.f;
#pragma unroll
      for (int i = qk; i < ks; i += 4) {
        const float* zr = sm + L.b_at(L.z, rk - i + kc, ck + kc);
        const float* kr = sm + L.kern + i * ks;
#pragma unroll
        for (int j = 0; j < ks; ++j) s = fmaf(kr[j], zr[-j], s);
      }
      s = ts_sum4(s);
      if (qk == 0) ts_put_blur<P>(sm, L, L.rb, rk, ck, s - sm[L.y + pk], rank, base);
    }
    ts_cluster_arrive();  // [S1] rb halos published
    for (int t = threadIdx.x; t < (R + 2) * W * 4; t += TS_T) {
      const int p = t % ((R + 2) * W), q = t / ((R + 2) * W);
      const int r = p / W - 1, c = p % W;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const bool inside = row0 + r >= 0 && row0 + r < H;
      if (inside) {
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const int gr = row0 + r + tap / 3 - 1, cc = c + tap % 3 - 1;
          const float v = (gr >= 0 && gr < H && cc >= 0 && cc < W) ? sm[L.b_at(L.z, r + tap / 3 - 1, cc)] : 0.f;
          const float4 w = *reinterpret_cast<const float4*>(sm + L.w1f + tap * TS_C + 4 * q);
          acc[0] = fmaf(w.x, v, acc[0]); acc[1] = fmaf(w.y, v, acc[1]);
          acc[2] = fmaf(w.z, v, acc[2]); acc[3] = fmaf(w.w, v, acc[3]);
        }
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) sm[L.n_at(L.a1, 4 * q + e, r, c)] = inside ? ts_softplus(acc[e]) : 0.f;
    }
    __syncthreads();  // a1 was written after this CTA's arrive: the barrier does not order it
    TS_MARK(1)
    ts_cluster_wait();  // [S1] rb halos complete
    TS_MARK(2)
    // [2] a2 = sp(c2(a1)) (blocked threads, split over the input channels), pushed with a 2-row
    //     halo. The K parts' partial sums meet in shared memory and every output is their sum in
    //     the fixed order part 0 + part 1 + ...
    float acc[2][4];
    ts_conv16<false>(sm, L, L.a1, L.w2f, rb0, cb, qb, ci0, nci, acc);
#pragma unroll
    for (int i = 0; i < 8; ++i) sm[L.part + (kh * 8 + i) * nb + tb] = acc[i >> 2][i & 3];
    __syncthreads();
    for (int j = 0; j < nout; ++j) {
      const int i = kh * nout + j;
      float s = sm[L.part + i * nb + tb];
      for (int h = 1; h < ksplit; ++h) s += sm[L.part + (h * 8 + i) * nb + tb];
      ts_put_net(sm, L, L.n_at(L.a2, 4 * qb + (i & 3), rb0 + (i >> 2), cb), ts_softplus(s), rb0 + (i >> 2), rank, H,
                 2, base);
    }
    TS_MARK(3)
    ts_cluster_sync();  // [S2] a2 halos (2 rows)
    TS_MARK(4)
    // [3] U = c3(a2) on rows -1 .. R (zero outside the image): the identity skip makes grad g =
    //     J_U^T U (cotangent U); 4 lanes per pixel over the input channels
    for (int t = threadIdx.x; t < (R + 2) * W * 4; t += TS_T) {
      const int p = t >> 2, q = t & 3, r = p / W - 1, c = p % W;
      float s = 0.f;
#pragma unroll
      for (int cj = 0; cj < TS_C / 4; ++cj) {
        const int ci = 4 * q + cj;
        const float* in = sm + L.n_at(L.a2, ci, r, c);
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) s = fmaf(sm[L.w3f + ci * 9 + tap], in[(tap / 3 - 1) * L.WP + tap % 3 - 1], s);
      }
      s = ts_sum4(s);
      if (q == 0) sm[L.n_at(L.u, 0, r, c)] = (row0 + r >= 0 && row0 + r < H) ? s : 0.f;
    }
    __syncthreads();
    // [4] q2 = c3^T(U) . sp'(a2)   (conv3x3^T: flipped taps), pushed (1-row halo);
    //     gf = A^T rb on the threads past the q2 items (rb is complete since [S1] and unchanged
    //     until the next iteration's [1]; gf is read in [6])
    for (int t = threadIdx.x; t < RW * 6; t += TS_T) {
      if (t >= RW * 4) {  // warp-uniform (RW is a multiple of 32): 2 lanes per pixel,
                          // (A^T rb)[r][c] = sum k[i][j] rb[r + i - kc][c + j - kc]
        const int u = t - RW * 4, p = u >> 1, h = u & 1, r = p / W, c = p % W;
        float s = 0.f;
#pragma unroll
        for (int i = h; i < ks; i += 2) {
          const float* rr = sm + L.b_at(L.rb, r + i - kc, c - kc);
          const float* kr = sm + L.kern + i * ks;
#pragma unroll
          for (int j = 0; j < ks; ++j) s = fmaf(kr[j], rr[j], s);
        }
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        if (h == 0) sm[L.gf + p] = s;
        continue;
      }
      const int p = t % RW, q = t / RW, r = p / W, c = p % W;
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
      const float* in = sm + L.n_at(L.u, 0, r, c);
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        const float v = in[(1 - tap / 3) * L.WP + 1 - tap % 3];
        const float4 w = *reinterpret_cast<const float4*>(sm + L.w3t + tap * TS_C + 4 * q);
        acc[0] = fmaf(w.x, v, acc[0]); acc[1] = fmaf(w.y, v, acc[1]);
        acc[2] = fmaf(w.z, v, acc[2]); acc[3] = fmaf(w.w, v, acc[3]);
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int o = L.n_at(0, 4 * q + e, r, c);
        ts_put_net(sm, L, L.q2 + o, acc[e] * ts_dsp(sm[L.a2 + o]), r, rank, H, 1, base);
      }
    }
    TS_MARK(5)
    ts_cluster_sync();  // [S3] q2 halos
    TS_MARK(6)
    // [5] q1 = c2^T(q2) . sp'(a1) (blocked threads, split as in [2]), pushed (1-row halo)
    ts_conv16<true>(sm, L, L.q2, L.w2t, rb0, cb, qb, ci0, nci, acc);
#pragma unroll
    for (int i = 0; i < 8; ++i) sm[L.part + (kh * 8 + i) * nb + tb] = acc[i >> 2][i & 3];
    __syncthreads();
    for (int j = 0; j < nout; ++j) {
      const int i = kh * nout + j;
      float s = sm[L.part + i * nb + tb];
      for (int h = 1; h < ksplit; ++h) s += sm[L.part + (h * 8 + i) * nb + tb];
      const int o = L.n_at(0, 4 * qb + (i & 3), rb0 + (i >> 2), cb);
      ts_put_net(sm, L, L.q1 + o, s * ts_dsp(sm[L.a1 + o]), rb0 + (i >> 2), rank, H, 1, base);
    }
    TS_MARK(7)
    ts_cluster_sync();  // [S4] q1 halos
    TS_MARK(8)
    // [6] grad g = c1^T(q1); x^{k+1} = z - tau (grad f + lam grad g) (Alg. 1 l.8); residual partials
    float d2 = 0.f, n2 = 0.f, bad = 0.f;
    if (act_k) {
      float s = 0.f;
#pragma unroll
      for (int cj = 0; cj < TS_C / 4; ++cj) {
        const int co = 4 * qk + cj;
        const float* in = sm + L.n_at(L.q1, co, rk, ck);
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) s = fmaf(sm[L.w1t + co * 9 + tap], in[(1 - tap / 3) * L.WP + 1 - tap % 3], s);
      }
      s = ts_sum4(s);
      if (qk == 0) {
        const float z = sm[L.b_at(L.z, rk, ck)], xk = sm[xk_o + pk];
        const float x1 = z - A.tau * (sm[L.gf + pk] + A.lam * s);
        sm[xn_o + pk] = x1;  // candidate x^{k+1}
        const float d = x1 - xk;
        if (isfinite(x1)) d2 = d * d; else bad = 1.f;
        n2 = xk * xk;
        // candidate z^{k+1} = x^{k+1} + beta (x^{k+1} - x^k) (Eq. 4), pushed now so that the
        // residual's barrier also completes the next iteration's z halos (every read of z^k by
        // a neighbour happened before [S1]; a diverged or converged image exits before using it)
        ts_put_blur<P>(sm, L, L.z, rk, ck, x1 + A.beta * (x1 - xk), rank, base);
      }
    }
    // block reduction (fixed order), then this CTA's partials into slot `rank` of every CTA
    {
      __shared__ float wred[3][TS_T / 32];
      const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        d2 += __shfl_xor_sync(0xffffffffu, d2, o);
        n2 += __shfl_xor_sync(0xffffffffu, n2, o);
        bad += __shfl_xor_sync(0xffffffffu, bad, o);
      }
      if (lane == 0) { wred[0][wid] = d2; wred[1][wid] = n2; wred[2][wid] = bad; }
      __syncthreads();
      if (threadIdx.x < P) {
        float a = 0.f, b = 0.f, e = 0.f;
        for (int w = 0; w < TS_T / 32; ++w) { a += wred[0][w]; b += wred[1][w]; e += wred[2][w]; }
        const uint32_t dst = ts_mapa(base + 4u * (uint32_t)(L.red + rank * 4), (uint32_t)threadIdx.x);
        ts_st_cluster(dst, a);
        ts_st_cluster(dst + 4, b);
        ts_st_cluster(dst + 8, e);
      }
    }
    TS_MARK(9)
    ts_cluster_sync();  // [S5] partials, z^{k+1}
    TS_MARK(10)
    // the P partials in fp64, summed by every warp with the same butterfly (a + b = b + a, so every
    // lane, warp and CTA gets the identical value: one stop decision for the cluster)
    double D2 = 0.0, N2 = 0.0, BAD = 0.0;
    {
      const int ln = threadIdx.x & 31;
      if (ln < P) {
        D2 = (double)sm[L.red + ln * 4];
        N2 = (double)sm[L.red + ln * 4 + 1];
        BAD = (double)sm[L.red + ln * 4 + 2];
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        D2 += __shfl_xor_sync(0xffffffffu, D2, o);
        N2 += __shfl_xor_sync(0xffffffffu, N2, o);
        BAD += __shfl_xor_sync(0xffffffffu, BAD, o);
      }
    }
    if (BAD > 0.0 || !isfinite(D2)) {  // reading Q22: keep x^k, status diverged
      status = 2;
      break;
    }
    res = N2 > 0.0 ? sqrtf((float)D2) / sqrtf((float)N2) : INFINITY;  // fp64 sums, fp32 root (res is fp32)
    iters = k + 1;
    // accept: x^k <- x^{k+1} (z^{k+1} is already in place)
    { const int t = xk_o; xk_o = xn_o; xn_o = t; }  // x^k <- x^{k+1}: the planes swap roles
    if (rank == 0 && threadIdx.x == 0 && A.trace && k < A.trace_cap)
      atomicMax(reinterpret_cast<int*>(A.trace) + k, __float_as_int(res));
    TS_MARK(11)
    if (((k + 1) % A.check_every) == 0 && res <= A.tol) {
      status = 0;
      break;
    }
  }
  // x-hat = the last accepted iterate (Remark 1)
  __syncthreads();
  for (int t = threadIdx.x; t < RW; t += TS_T) A.x[img + t] = sm[xk_o + t];
  if (rank == 0 && threadIdx.x == 0) {
    A.iters[n] = iters;
    A.res[n] = res;
    A.status[n] = status;
    atomicMax(A.kdone, iters);
  }
  ts_cluster_sync();  // no CTA exits while a neighbour may still write into its shared memory
}

// cluster size for an image of H rows: 16 CTAs (2 rows each) where that fits, else 8
static int ts_cluster(int H) { return (H % 16 == 0 && (H / 16) % 2 == 0) ? 16 : 8; }

size_t tiny_solve_smem(int H, int W, int ks) {
  TsLayout L;
  L.init(H / ts_cluster(H), W, ks);
  return sizeof(float) * (size_t)L.total;
}

// (R + 2) W x 4 items per recomputed stage are looped; R x W <= 128 keeps one pixel per 4 lanes
bool tiny_solve_supported(int H, int W, int ks) {
  const int P = ts_cluster(H);
  if (H % P != 0 || W % 32 != 0 || W < ks) return false;
  const int R = H / P;
  const int HB = (ks - 1) / 2 > 1 ? (ks - 1) / 2 : 1;
  // 4 lanes per pixel, whole warps per stage, 2-row blocks; the blur halo (HB rows) within the
  // image and the network halos (2 rows) from the adjacent CTAs
  if (R * W > TS_T / 4 || R % 2 != 0 || R < 2 || HB > (P / 2) * R) return false;
  return tiny_solve_smem(H, W, ks) <= 200 * 1024;
}

template <int P, int KS>
static void launch_tiny_p(const TinyArgs& A, size_t smem, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(P * A.N));
  cfg.blockDim = dim3(TS_T);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, tiny_solve_kernel<P, KS>, A);
}

void launch_tiny_solve(const TinySolveArgs& a, cudaStream_t s) {
  TinyArgs A{};
  const int P = ts_cluster(a.H);
  A.N = a.N; A.H = a.H; A.W = a.W; A.R = a.H / P;
  A.ks = a.ks; A.kper = a.kper; A.kern = a.kern;
  A.w1 = a.w1; A.w2 = a.w2; A.w3 = a.w3; A.y = a.y; A.x = a.x;
  A.lam = a.lam; A.tau = a.tau; A.beta = a.beta; A.tol = a.tol;
  A.max_iter = a.max_iter; A.check_every = a.check_every;
  A.iters = a.iters; A.res = a.res; A.status = a.status; A.trace = a.trace; A.trace_cap = a.trace_cap;
  A.kdone = a.kdone;
  const size_t smem = tiny_solve_smem(a.H, a.W, a.ks);
  if (P == 16) {
    if (a.ks == 9) launch_tiny_p<16, 9>(A, smem, s);
    else launch_tiny_p<16, 0>(A, smem, s);
  } else {
    if (a.ks == 9) launch_tiny_p<8, 9>(A, smem, s);
    else launch_tiny_p<8, 0>(A, smem, s);
  }
}

void init_attrs_tiny() {
  set_max_dyn_smem(tiny_solve_kernel<8, 0>);
  set_max_dyn_smem(tiny_solve_kernel<8, 9>);
  set_max_dyn_smem(tiny_solve_kernel<16, 0>);
  set_max_dyn_smem(tiny_solve_kernel<16, 9>);
  cudaFuncSetAttribute(tiny_solve_kernel<16, 0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  cudaFuncSetAttribute(tiny_solve_kernel<16, 9>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
}

}  // namespace ideq
