// Whole-solve persistent kernel for the tiny network of BASELINE config C1 (1 x 32 x 32 image,
// N(x) = x + c3(sp(c2(sp(c1(x))))), widths 1 -> 16 -> 16 -> 1, periodic blur, gradient step):
// the i-DEQ loop of Alg. 1 -- extrapolation (Eq. 4), the network and
// its input VJP (Eq. 2), the fidelity gradient A^T(Az - y), the update (Alg. 1 l.8,
// P:219), the residual ||x^{k+1} - x^k|| / ||x^k|| and the stop rule -- runs for all
// iterations inside ONE launch. The per-iteration path costs ~11 launches (72 us per iteration,
// launch- and latency-bound); here every operand stays in shared memory.
//
// One image = one thread-block cluster of 8 CTAs (a batch runs one cluster per image). CTA r owns
// rows [r R, (r + 1) R) of the image (R = H / 8) and keeps every tensor of the iteration for those
// rows plus a halo of HB rows above and below: z, the blur residual, U, and the 16-channel
// activations a1, a2 and cotangents q2, q1. After each stage the CTAs meet at a cluster barrier
// and copy the halo rows they need from their neighbours' shared memory (DSMEM). The residual's
// three partial sums are written into every CTA's shared memory and combined in fp64 in a fixed
// order, so all 8 CTAs take the identical stop decision without a second barrier.
//
// fp32 throughout (the FFMA path's arithmetic: exact fp32 softplus / sigmoid), matching the fp32
// parity mode. Supported: TINY3 with hidden width 16, C = 1, identity skip, softplus, direct blur
// gradient step, per-image stop rule, no restart / averaging (the runtime falls back otherwise).
#include "common.cuh"
#include "kernels.h"

namespace ideq {

constexpr int TS_P = 8;          // CTAs per image (cluster size)
constexpr int TS_T = 256;        // threads per CTA
constexpr int TS_C = 16;         // hidden width

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
__device__ __forceinline__ void ts_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t ts_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// Shared-memory layout (floats): halo planes hold rows -HB .. R+HB-1 of one channel, PL = (R+2HB) W.
struct TsLayout {
  int R, W, HB, PL;
  int z, rb, u, a1, a2, q2, q1;    // halo planes (a1..q1: 16 channels each)
  int xk, gf, gg, y;               // own-row planes (R W)
  int w1f, w2f, w3f, w1t, w2t, w3t, kern, red;
  int total;
  __host__ __device__ void init(int R_, int W_, int HB_, int ks) {
    R = R_; W = W_; HB = HB_;
    PL = (R + 2 * HB) * W;
    int o = 0;
    auto take = [&](int n) { const int b = o; o += (n + 3) & ~3; return b; };
    z = take(PL); rb = take(PL); u = take(PL);
    a1 = take(TS_C * PL); a2 = take(TS_C * PL); q2 = take(TS_C * PL); q1 = take(TS_C * PL);
    xk = take(R * W); gf = take(R * W); gg = take(R * W); y = take(R * W);
    w1f = take(9 * TS_C); w2f = take(TS_C * 9 * TS_C); w3f = take(TS_C * 9);
    w1t = take(TS_C * 9); w2t = take(TS_C * 9 * TS_C); w3t = take(9 * TS_C);
    kern = take(ks * ks); red = take(TS_P * 4);
    total = o;
  }
};

struct TinyArgs {
  int N, H, W, R, HB, ks, kper;
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

// Copy rows [-h, -1] and [R, R + h - 1] of `nch` halo planes starting at smem float offset `off`
// from the owners' shared memory (periodic in the image row; conv stages mask rows outside the
// image themselves).
__device__ __forceinline__ void ts_halo(float* sm, const TsLayout& L, int off, int nch, int h, int row0, int H) {
  const uint32_t base = ts_smem_u32(sm);
  const int per = 2 * h * L.W;
  for (int t = threadIdx.x; t < nch * per; t += TS_T) {
    const int ch = t / per, q = t % per;
    const int rr = q / L.W, c = q % L.W;
    const int r = rr < h ? rr - h : L.R + (rr - h);  // local row
    int gr = row0 + r;
    gr = ((gr % H) + H) % H;
    const uint32_t src_cta = (uint32_t)(gr / L.R), src_row = (uint32_t)(gr % L.R);
    const int src = off + ch * L.PL + (int)(src_row + L.HB) * L.W + c;
    sm[off + ch * L.PL + (r + L.HB) * L.W + c] = ts_ld_cluster(ts_mapa(base + 4u * (uint32_t)src, src_cta));
  }
}

__device__ __forceinline__ float ts_softplus(float t) { return fmaxf(t, 0.f) + log1pf(__expf(-fabsf(t))); }
__device__ __forceinline__ float ts_dsp(float a) { return -expm1f(-a); }  // sigmoid(p) from a = sp(p)

// in-plane value with the conv's zero padding: local row r (may be in the halo), column c
__device__ __forceinline__ float ts_at(const float* p, const TsLayout& L, int r, int c, int row0, int H) {
  const int gr = row0 + r;
  if (gr < 0 || gr >= H || c < 0 || c >= L.W) return 0.f;
  return p[(r + L.HB) * L.W + c];
}

__global__ void __cluster_dims__(TS_P, 1, 1) __launch_bounds__(TS_T, 1) tiny_solve_kernel(TinyArgs A) {
  extern __shared__ __align__(16) float sm[];
  const int rank = (int)ts_rank();
  const int n = blockIdx.x / TS_P;
  const int H = A.H, W = A.W, R = A.R;
  const int row0 = rank * R;
  TsLayout L;
  L.init(R, W, A.HB, A.ks);
  const int RW = R * W;
  const int kc = (A.ks - 1) / 2;
  // ---- weights (fwd layouts [tap][co] / [ci][tap][co]; adjoint layouts over the input channel)
  for (int t = threadIdx.x; t < 9 * TS_C; t += TS_T) {
    const int co = t / 9, tap = t % 9;
    sm[L.w1f + tap * TS_C + co] = A.w1[co * 9 + tap];  // c1 [co][0][tap]
    sm[L.w1t + co * 9 + tap] = A.w1[co * 9 + tap];     // c1^T: [co][tap]
    sm[L.w3f + co * 9 + tap] = A.w3[co * 9 + tap];     // c3 [0][ci = co][tap]
    sm[L.w3t + tap * TS_C + co] = A.w3[co * 9 + tap];  // c3^T: [tap][ci]
  }
  for (int t = threadIdx.x; t < TS_C * TS_C * 9; t += TS_T) {
    const int co = t / (TS_C * 9), ci = (t / 9) % TS_C, tap = t % 9;
    sm[L.w2f + (ci * 9 + tap) * TS_C + co] = A.w2[t];  // c2: [ci][tap][co]
    sm[L.w2t + (co * 9 + tap) * TS_C + ci] = A.w2[t];  // c2^T: [co][tap][ci]
  }
  const float* kg = A.kern + (A.kper ? (long long)n * A.ks * A.ks : 0);
  for (int t = threadIdx.x; t < A.ks * A.ks; t += TS_T) sm[L.kern + t] = kg[t];
  // ---- state: x^0 (own rows), z^0 = x^0, y
  const long long img = (long long)n * H * W;
  for (int t = threadIdx.x; t < RW; t += TS_T) {
    const float v = A.x[img + (long long)row0 * W + t];
    sm[L.xk + t] = v;
    sm[L.z + L.HB * W + t] = v;
    sm[L.y + t] = A.y[img + (long long)row0 * W + t];
  }
  int iters = 0, status = 1;
  float res = __int_as_float(0x7fc00000);
  __syncthreads();
  for (int k = 0; k < A.max_iter; ++k) {
    // [S0] z complete on every CTA: halo rows (+-HB, periodic: the blur reads them wrapped)
    ts_cluster_sync();
    ts_halo(sm, L, L.z, 1, L.HB, row0, H);
    __syncthreads();
    // [1] a1 = sp(c1(z)); blur residual rb = A z - y (true periodic convolution, reading Q8)
    for (int t = threadIdx.x; t < RW; t += TS_T) {
      const int r = t / W, c = t % W;
      float acc[TS_C];
#pragma unroll
      for (int co = 0; co < TS_C; ++co) acc[co] = 0.f;
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        const float v = ts_at(sm + L.z, L, r + tap / 3 - 1, c + tap % 3 - 1, row0, H);
        const float4* w4 = reinterpret_cast<const float4*>(sm + L.w1f + tap * TS_C);
#pragma unroll
        for (int q = 0; q < TS_C / 4; ++q) {
          const float4 w = w4[q];
          acc[4 * q] = fmaf(w.x, v, acc[4 * q]);
          acc[4 * q + 1] = fmaf(w.y, v, acc[4 * q + 1]);
          acc[4 * q + 2] = fmaf(w.z, v, acc[4 * q + 2]);
          acc[4 * q + 3] = fmaf(w.w, v, acc[4 * q + 3]);
        }
      }
#pragma unroll
      for (int co = 0; co < TS_C; ++co) sm[L.a1 + co * L.PL + (r + L.HB) * W + c] = ts_softplus(acc[co]);
      float s = 0.f;
      for (int i = 0; i < A.ks; ++i) {
        const float* zr = sm + L.z + (r - i + kc + L.HB) * W;
        for (int j = 0; j < A.ks; ++j) {
          int cc = c - j + kc;
          cc = cc < 0 ? cc + W : (cc >= W ? cc - W : cc);
          s = fmaf(sm[L.kern + i * A.ks + j], zr[cc], s);
        }
      }
      sm[L.rb + (r + L.HB) * W + c] = s - sm[L.y + t];
    }
    // [S1] a1 (+-1) and rb (+-HB) halos
    ts_cluster_sync();
    ts_halo(sm, L, L.a1, TS_C, 1, row0, H);
    ts_halo(sm, L, L.rb, 1, L.HB, row0, H);
    __syncthreads();
    // [2] a2 = sp(c2(a1)) (thread = pixel x half of the output channels); gf = A^T rb
    for (int t = threadIdx.x; t < 2 * RW; t += TS_T) {
      const int p = t % RW, half = t / RW;
      const int r = p / W, c = p % W;
      float acc[TS_C / 2];
#pragma unroll
      for (int co = 0; co < TS_C / 2; ++co) acc[co] = 0.f;
      for (int ci = 0; ci < TS_C; ++ci) {
        const float* in = sm + L.a1 + ci * L.PL;
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const float v = ts_at(in, L, r + tap / 3 - 1, c + tap % 3 - 1, row0, H);
          const float4* w4 = reinterpret_cast<const float4*>(sm + L.w2f + (ci * 9 + tap) * TS_C + half * (TS_C / 2));
#pragma unroll
          for (int q = 0; q < TS_C / 8; ++q) {
            const float4 w = w4[q];
            acc[4 * q] = fmaf(w.x, v, acc[4 * q]);
            acc[4 * q + 1] = fmaf(w.y, v, acc[4 * q + 1]);
            acc[4 * q + 2] = fmaf(w.z, v, acc[4 * q + 2]);
            acc[4 * q + 3] = fmaf(w.w, v, acc[4 * q + 3]);
          }
        }
      }
#pragma unroll
      for (int co = 0; co < TS_C / 2; ++co)
        sm[L.a2 + (half * (TS_C / 2) + co) * L.PL + (r + L.HB) * W + c] = ts_softplus(acc[co]);
      if (half == 0) {  // (A^T rb)[r][c] = sum_ij k[i][j] rb[r + i - kc][(c + j - kc) mod W]   (correlation)
        float s = 0.f;
        for (int i = 0; i < A.ks; ++i) {
          const float* rr = sm + L.rb + (r + i - kc + L.HB) * W;
          for (int j = 0; j < A.ks; ++j) {
            int cc = c + j - kc;
            cc = cc < 0 ? cc + W : (cc >= W ? cc - W : cc);
            s = fmaf(sm[L.kern + i * A.ks + j], rr[cc], s);
          }
        }
        sm[L.gf + p] = s;
      }
    }
    // [S2] a2 halo
    ts_cluster_sync();
    ts_halo(sm, L, L.a2, TS_C, 1, row0, H);
    __syncthreads();
    // [3] U = c3(a2): with the identity skip N(z) = z + U, grad g = J_U^T U (cotangent U)
    for (int t = threadIdx.x; t < RW; t += TS_T) {
      const int r = t / W, c = t % W;
      float s = 0.f;
      for (int ci = 0; ci < TS_C; ++ci) {
        const float* in = sm + L.a2 + ci * L.PL;
#pragma unroll
        for (int tap = 0; tap < 9; ++tap)
          s = fmaf(sm[L.w3f + ci * 9 + tap], ts_at(in, L, r + tap / 3 - 1, c + tap % 3 - 1, row0, H), s);
      }
      sm[L.u + (r + L.HB) * W + c] = s;
    }
    ts_cluster_sync();
    ts_halo(sm, L, L.u, 1, 1, row0, H);
    __syncthreads();
    // [4] q2 = c3^T(U) . sp'(a2)   (conv3x3^T: flipped taps)
    for (int t = threadIdx.x; t < RW; t += TS_T) {
      const int r = t / W, c = t % W;
      float acc[TS_C];
#pragma unroll
      for (int ci = 0; ci < TS_C; ++ci) acc[ci] = 0.f;
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        const float v = ts_at(sm + L.u, L, r + 1 - tap / 3, c + 1 - tap % 3, row0, H);
        const float4* w4 = reinterpret_cast<const float4*>(sm + L.w3t + tap * TS_C);
#pragma unroll
        for (int q = 0; q < TS_C / 4; ++q) {
          const float4 w = w4[q];
          acc[4 * q] = fmaf(w.x, v, acc[4 * q]);
          acc[4 * q + 1] = fmaf(w.y, v, acc[4 * q + 1]);
          acc[4 * q + 2] = fmaf(w.z, v, acc[4 * q + 2]);
          acc[4 * q + 3] = fmaf(w.w, v, acc[4 * q + 3]);
        }
      }
#pragma unroll
      for (int ci = 0; ci < TS_C; ++ci) {
        const int o = ci * L.PL + (r + L.HB) * W + c;
        sm[L.q2 + o] = acc[ci] * ts_dsp(sm[L.a2 + o]);
      }
    }
    ts_cluster_sync();
    ts_halo(sm, L, L.q2, TS_C, 1, row0, H);
    __syncthreads();
    // [5] q1 = c2^T(q2) . sp'(a1)
    for (int t = threadIdx.x; t < 2 * RW; t += TS_T) {
      const int p = t % RW, half = t / RW;
      const int r = p / W, c = p % W;
      float acc[TS_C / 2];
#pragma unroll
      for (int ci = 0; ci < TS_C / 2; ++ci) acc[ci] = 0.f;
      for (int co = 0; co < TS_C; ++co) {
        const float* in = sm + L.q2 + co * L.PL;
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const float v = ts_at(in, L, r + 1 - tap / 3, c + 1 - tap % 3, row0, H);
          const float4* w4 = reinterpret_cast<const float4*>(sm + L.w2t + (co * 9 + tap) * TS_C + half * (TS_C / 2));
#pragma unroll
          for (int q = 0; q < TS_C / 8; ++q) {
            const float4 w = w4[q];
            acc[4 * q] = fmaf(w.x, v, acc[4 * q]);
            acc[4 * q + 1] = fmaf(w.y, v, acc[4 * q + 1]);
            acc[4 * q + 2] = fmaf(w.z, v, acc[4 * q + 2]);
            acc[4 * q + 3] = fmaf(w.w, v, acc[4 * q + 3]);
          }
        }
      }
#pragma unroll
      for (int ci = 0; ci < TS_C / 2; ++ci) {
        const int o = (half * (TS_C / 2) + ci) * L.PL + (r + L.HB) * W + c;
        sm[L.q1 + o] = acc[ci] * ts_dsp(sm[L.a1 + o]);
      }
    }
    ts_cluster_sync();
    ts_halo(sm, L, L.q1, TS_C, 1, row0, H);
    __syncthreads();
    // [6] grad g = c1^T(q1); x^{k+1} = z - tau (grad f + lam grad g) (Alg. 1 l.8); residual partials
    float d2 = 0.f, n2 = 0.f, bad = 0.f;
    for (int t = threadIdx.x; t < RW; t += TS_T) {
      const int r = t / W, c = t % W;
      float s = 0.f;
      for (int co = 0; co < TS_C; ++co) {
        const float* in = sm + L.q1 + co * L.PL;
#pragma unroll
        for (int tap = 0; tap < 9; ++tap)
          s = fmaf(sm[L.w1t + co * 9 + tap], ts_at(in, L, r + 1 - tap / 3, c + 1 - tap % 3, row0, H), s);
      }
      const float z = sm[L.z + (r + L.HB) * W + c], xk = sm[L.xk + t];
      const float x1 = z - A.tau * (sm[L.gf + t] + A.lam * s);
      sm[L.gg + t] = x1;  // candidate x^{k+1}
      const float d = x1 - xk;
      if (isfinite(x1)) d2 += d * d; else bad += 1.f;
      n2 += xk * xk;
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
      if (threadIdx.x < TS_P) {
        float a = 0.f, b = 0.f, e = 0.f;
        for (int w = 0; w < TS_T / 32; ++w) { a += wred[0][w]; b += wred[1][w]; e += wred[2][w]; }
        const uint32_t slot = ts_smem_u32(sm + L.red + rank * 4);
        const uint32_t dst = ts_mapa(slot, (uint32_t)threadIdx.x);
        ts_st_cluster(dst, a);
        ts_st_cluster(dst + 4, b);
        ts_st_cluster(dst + 8, e);
      }
    }
    ts_cluster_sync();
    double D2 = 0.0, N2 = 0.0, BAD = 0.0;
    for (int q = 0; q < TS_P; ++q) {  // fixed order: identical on every CTA
      D2 += (double)sm[L.red + q * 4];
      N2 += (double)sm[L.red + q * 4 + 1];
      BAD += (double)sm[L.red + q * 4 + 2];
    }
    if (BAD > 0.0 || !isfinite(D2)) {  // reading Q22: keep x^k, status diverged
      status = 2;
      break;
    }
    const double rr = N2 > 0.0 ? sqrt(D2) / sqrt(N2) : (double)INFINITY;
    res = (float)rr;
    iters = k + 1;
    // accept: z^{k+1} = x^{k+1} + beta (x^{k+1} - x^k) (Eq. 4), x^k <- x^{k+1}
    for (int t = threadIdx.x; t < RW; t += TS_T) {
      const float x1 = sm[L.gg + t], xk = sm[L.xk + t];
      sm[L.z + L.HB * W + t] = x1 + A.beta * (x1 - xk);
      sm[L.xk + t] = x1;
    }
    if (rank == 0 && threadIdx.x == 0 && A.trace && k < A.trace_cap)
      atomicMax(reinterpret_cast<int*>(A.trace) + k, __float_as_int(res));
    if (((k + 1) % A.check_every) == 0 && res <= A.tol) {
      status = 0;
      break;
    }
    __syncthreads();
  }
  // x-hat = the last accepted iterate (Remark 1)
  __syncthreads();
  for (int t = threadIdx.x; t < RW; t += TS_T) A.x[img + (long long)row0 * W + t] = sm[L.xk + t];
  if (rank == 0 && threadIdx.x == 0) {
    A.iters[n] = iters;
    A.res[n] = res;
    A.status[n] = status;
    atomicMax(A.kdone, iters);
  }
  ts_cluster_sync();  // no CTA exits while a neighbour may still read its shared memory
}

size_t tiny_solve_smem(int H, int W, int ks) {
  TsLayout L;
  L.init(H / TS_P, W, (ks - 1) / 2 > 1 ? (ks - 1) / 2 : 1, ks);
  return sizeof(float) * (size_t)L.total;
}

bool tiny_solve_supported(int H, int W, int ks) {
  if (H % TS_P != 0 || (H / TS_P) < (ks - 1) / 2 || W < ks || W > 128) return false;
  return tiny_solve_smem(H, W, ks) <= 200 * 1024;
}

void launch_tiny_solve(const TinySolveArgs& a, cudaStream_t s) {
  TinyArgs A{};
  A.N = a.N; A.H = a.H; A.W = a.W; A.R = a.H / TS_P;
  A.HB = (a.ks - 1) / 2 > 1 ? (a.ks - 1) / 2 : 1;
  A.ks = a.ks; A.kper = a.kper; A.kern = a.kern;
  A.w1 = a.w1; A.w2 = a.w2; A.w3 = a.w3; A.y = a.y; A.x = a.x;
  A.lam = a.lam; A.tau = a.tau; A.beta = a.beta; A.tol = a.tol;
  A.max_iter = a.max_iter; A.check_every = a.check_every;
  A.iters = a.iters; A.res = a.res; A.status = a.status; A.trace = a.trace; A.trace_cap = a.trace_cap;
  A.kdone = a.kdone;
  const size_t smem = tiny_solve_smem(a.H, a.W, a.ks);
  tiny_solve_kernel<<<dim3(TS_P * a.N), dim3(TS_T), smem, s>>>(A);
}

void init_attrs_tiny() { set_max_dyn_smem(tiny_solve_kernel); }

}  // namespace ideq
