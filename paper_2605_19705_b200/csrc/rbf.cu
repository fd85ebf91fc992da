// Residual-block-fused level-0 convolutions (bf16, tcgen05, row streaming).
//
// A residual block of the U-Net (reading Q10) is two 3x3 convolutions at the same width:
//   forward (Eq. 2's network):  a = sp(A t)  (saved for the VJP),  t' = t + B a
//   input VJP (its transpose):           q = (B^T g) . sp'(a),              g' = g + A^T q
// Run as two launches, the intermediate (a or q) makes a round trip through HBM and the block
// input is read twice (conv input, then residual): at level 0 of C3 that is 671 MB (forward) /
// 805 MB (VJP) per block for 403 MB of compulsory traffic. This kernel computes the whole block
// for full image rows:
//
//   * a CTA owns a run of consecutive output rows of one image and streams down it. Input rows x
//     (the block input t or g) arrive by TMA into a ring of full-width rows with a zero pixel on
//     either side (the zero padding in w); out-of-image rows are zero-filled by TMA (padding in h);
//   * stage 1 computes the intermediate rows u from x, stage 2 the output rows from u. Both fold
//     the kernel ROW into the GEMM's N dimension: input row r, for each kernel column dw (the A
//     operand shifted by dw pixels) and 16-channel K step, is ONE MMA of N = 96 whose three
//     32-column blocks are the output rows r+1, r, r-1 (taps dh = -1, 0, +1). Output rows are
//     accumulated in a ring of R TMEM blocks (a block is complete after its third input row) and
//     each input row is read from shared memory 3 times per convolution instead of 9 (the level-0
//     convolutions, N = 32, are otherwise bound by the shared-memory operand path). A window that
//     wraps around the ring is issued as two MMAs. The epilogue zeroes a block after reading it,
//     so every MMA accumulates;
//   * stage-1 epilogue: softplus (forward; also stored to HBM as the saved activation a) or the
//     sp'(a) product with the saved activation read from HBM (VJP), written in the UMMA operand
//     layout into a ring of u rows (rows outside the image are zeros: conv 2's padding in h);
//   * stage-2 epilogue: + the residual (the block input row, re-read from L2), stored with
//     16-byte global stores (the two warps of a 32-byte sector store it back to back).
// HBM traffic per block: read x (+ a in the VJP), write a (forward) and the output.
// Each run recomputes two intermediate rows (h0 - 1 and h1) and reads two extra input rows.
//
// Warp roles (one CTA per SM): warp 0 TMA producer, warp 1 TMEM allocator + MMA issuer, then
// 8 stage-1 epilogue warps per M tile (W = 256: warps 2..17, one tile each) and 8 stage-2
// epilogue warps for the whole row (each: TMEM lane quadrant = warp % 4, 16-channel half).
// MMA order per run: S1(k) for input rows k = 0 .. nu+1, and S2(j) for intermediate row j right
// after S1(j+3), so the stage-1 epilogue of row j overlaps two MMA stages before S2(j) reads it.
//
// Status (B200, C3 level 0, 32 x 256 x 256 x 32): in the solver's captured iteration the fused
// blocks take the C3 step from 3.41 to 3.33 ms in a same-box A/B (tools/rbf_ab.py) and the bench
// to 10.6k image-iterations/s, so the solver uses them by default (ideq_debug_set_fusion turns
// them off; tests/test_gpu_rbf.py checks both against the oracle and each other). Serialised and
// cold under ncu a block takes ~132 us against 131 / 136 us for the two unfused launches: the win
// is the halved HBM traffic overlapping the neighbours under programmatic dependent launch.
// What bounds it (tools/rbf_prof.cu stage timeline and its RBF_NO_MMA / RBF_NO_EPI bisection
// builds, ncu source-level stalls, tools/mma_rate_probe.cu):
//   * the MMA stream alone (epilogues reduced to their barrier arrivals) takes ~97 us per block,
//     the epilogues alone (no MMAs) ~101 us (forward) / ~135 us (VJP), the skeleton of barriers
//     and row loads ~43 us; together 139 / 142 us: the two halves overlap only partly, each
//     epilogue group waiting most of the time on the MMA commits and the MMA warp on the freed
//     ring blocks;
//   * the epilogue's fixed per-row latency: its proxy fence (MEMBAR.ALL.CTA) waits for every
//     outstanding global access of the thread. Hence the forward's saved activation goes out by
//     TMA from the u ring (157 -> 139 us) and the VJP's saved-activation rows are bulk-prefetched
//     into L2 three rows ahead (152 -> 142 us);
//   * TMEM holds a 4-row ring per stage and M tile at W = 256 (2 stages x 2 tiles x 4 x 32
//     columns = 512), so a wrapped window must wait until the epilogue has drained the block it
//     adds +0 to (issuing it as two MMAs instead measured 2-3% slower); the two epilogue stages
//     run in separate warp groups so neither waits for the other's rows.
#include <cuda.h>
#include <type_traits>
#include <stdio.h>
#include <string.h>
#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace ideq {

// Epilogue groups: stage 1 has 8 warps per M tile (one tile per warp: 2 per TMEM lane quadrant,
// 16 channels each), stage 2 has 8 warps for all tiles of a row.
constexpr int RBF_GROUP_WARPS = 8;
template <int MT>
constexpr int rbf_threads() { return (2 + RBF_GROUP_WARPS * MT + RBF_GROUP_WARPS) * 32; }
constexpr int RBF_C = 32;                 // channels (64-byte pixels, SW64)
constexpr uint32_t RBF_PIX = RBF_C * 2;
constexpr uint32_t RBF_WTAP = RBF_C * RBF_PIX;     // 2 KB: B operand of one tap (32 rows x 64 B)
// B operand of one convolution, per kernel column dw: 6 blocks of 32 rows [w0 w1 w2 Z w0 w1]
// (w = window position, Z = zeros), so a ring window that wraps (ring blocks 2,3,0 or 3,0,1) is ONE
// N = 128 MMA over all four blocks with B starting at block 2 or 1 -- the fourth block gets +0
constexpr uint32_t RBF_WGROUP = 6 * RBF_WTAP;      // 12 KB
constexpr uint32_t RBF_WCONV = 3 * RBF_WGROUP;     // 36 KB per convolution

template <int MT>
struct RbfCfg {  // MT = W / 128 M tiles per row
  static constexpr int W = MT * 128;
  static constexpr int R = 4;                          // TMEM ring blocks per stage and M tile
  static constexpr int XS = MT == 1 ? 6 : 4;           // input-row ring (one S1 each + prefetch)
  static constexpr int US = MT == 1 ? 6 : 4;           // intermediate-row ring
  // slot: 1 KB pad (pixel -1 = zero at its end), W pixels, pixel W = zero, rounded to 1 KB
  static constexpr uint32_t SLOT = (1024u + (uint32_t)(W + 1) * RBF_PIX + 1023u) & ~1023u;
  static size_t smem() { return 1024 + 2 * RBF_WCONV + (size_t)(XS + US) * SLOT + 512; }
};

struct RbfParams {
  int N, H, W;
  int dh1[9], dw1[9], dh2[9], dw2[9];
  const __nv_bfloat16* w1;    // [9][32][32] GEMM operand of conv 1 / conv 2 (gemm_weights layout)
  const __nv_bfloat16* w2;
  const __nv_bfloat16* x;     // [N][H][W][32] block input (the residual, re-read from L2)
  __nv_bfloat16* out;         // [N][H][W][32] block output
  __nv_bfloat16* act;         // saved activation a: written (forward) / read (VJP)
  const int* act_list;        // live-image list (null: every image)
  const int* n_act;
};

// 16-byte chunk j (8 channels) of pixel p in a row payload (the SW64 pattern TMA / UMMA use)
__device__ __forceinline__ uint32_t rbf_chunk(uint32_t payload, int p, int j) {
  return payload + (uint32_t)p * RBF_PIX + (uint32_t)((j ^ ((p >> 1) & 3)) << 4);
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
      : "memory");
}
// timing-only bisection switches (tools/rbf_prof.cu builds; results are garbage when set)
#ifndef RBF_NO_MMA
#define RBF_NO_MMA 0
#endif
#ifndef RBF_NO_EPI
#define RBF_NO_EPI 0
#endif
#ifndef RBF_TRACE
#define RBF_TRACE 0
#endif
#if RBF_TRACE  // stage timeline of CTA 0 (tools/rbf_prof.cu): one clock per (event, row)
__device__ long long g_rbf_trace[16][256];
#define RBF_EV(code, row)                                                   \
  do {                                                                      \
    if (blockIdx.x == 0 && (row) >= 0 && (row) < 256) g_rbf_trace[code][row] = clock64(); \
  } while (0)
#else
#define RBF_EV(code, row) \
  do {                    \
  } while (0)
#endif
// forward: the saved activation row leaves shared memory (the u ring slot, already in the act
// tensor's SW64 layout) by one TMA tensor store per row. Per-thread global stores made the next
// row's proxy fence (MEMBAR.ALL.CTA + FENCE.VIEW.ASYNC) wait for them to complete: 157 -> 139 us
// per forward block (tools/rbf_prof.cu)
__device__ __forceinline__ void tma_store_4d(uint32_t src, const CUtensorMap* map, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(src)
               : "memory");
}
// mbarrier wait that suspends the thread (up to the hint, in ns) instead of spinning: the 16
// epilogue warps wait most of the time, and spinning try_wait loops take issue slots from the
// MMA warp that shares their scheduler
// (a plain try_wait or a test_wait spin measured the same, tools/rbf_prof.cu)
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WS_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WS_%=;\n}\n" ::"r"(bar),
      "r"(parity), "r"(1000000u)
      : "memory");
}
// named barrier 1 over the stage-1 epilogue group
template <int MT>
__device__ __forceinline__ void rbf_epi_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(RBF_GROUP_WARPS * MT * 32) : "memory");
}
// tcgen05.ld / st of 8 columns (32 lanes x 32 bit)
__device__ __forceinline__ void tmem_ld8_nw(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_zero8(uint32_t taddr) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(taddr), "r"(0u)
               : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// The CTA's runs: rows [q0, q1) of the (live) row sequence q = image_index * H + h, cut at image
// boundaries. Every role walks the same sequence.
struct RbfRun { int n, h0, h1; };
__device__ __forceinline__ bool rbf_next_run(const RbfParams& P, int& q, int q1, RbfRun& run) {
  if (q >= q1) return false;
  const int li = q / P.H;
  const int h0 = q - li * P.H;
  const int end = min(q1, (li + 1) * P.H);
  run.n = P.act_list ? __ldg(P.act_list + li) : li;
  run.h0 = h0;
  run.h1 = h0 + (end - q);
  q = end;
  return true;
}

template <int MT, bool VJP>
__global__ void __launch_bounds__(rbf_threads<MT>(), 1)
    rbf_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmAct,
               const __grid_constant__ RbfParams P) {
  using Cfg = RbfCfg<MT>;
  constexpr int XS = Cfg::XS, US = Cfg::US, R = Cfg::R, W = Cfg::W;
  constexpr uint32_t SLOT = Cfg::SLOT;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
  // [B operands conv 1 | conv 2][x ring][u ring][barriers]
  const uint32_t sW1 = base, sW2 = base + RBF_WCONV;
  const uint32_t sX = base + 2 * RBF_WCONV;
  const uint32_t sU = sX + XS * SLOT;
  const uint32_t sBar = sU + US * SLOT;
  const uint32_t xfull0 = sBar, xempty0 = xfull0 + 8u * XS, ufull0 = xempty0 + 8u * XS, uempty0 = ufull0 + 8u * US,
                 t1done0 = uempty0 + 8u * US, t1free0 = t1done0 + 8u * R, t2done0 = t1free0 + 8u * R,
                 t2free0 = t2done0 + 8u * R;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(gbase + (t2free0 + 8u * R - base));
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ---- prologue: B operands, grouped by kernel column dw: 3 groups of 6 blocks [w0 w1 w2 Z w0 w1]
  // of 32 rows (co), window position w = 0, 1, 2 <-> tap dh = +1, 0, -1 (the output rows r-1, r,
  // r+1 of input row r); K-major 64-byte rows, SW64. Zero rings (pad pixels stay zero), barriers,
  // TMEM.
  for (int i = threadIdx.x; i < 2 * 3 * 6 * RBF_C * 4; i += blockDim.x) {
    const int which = i / (18 * RBF_C * 4), rem = i % (18 * RBF_C * 4), row = rem >> 2, j = rem & 3;
    const int blk = (row / RBF_C) % 6, wpos = blk < 3 ? blk : (blk == 3 ? -1 : blk - 4);
    const int dwi = row / (6 * RBF_C) - 1, dh = wpos < 0 ? 99 : 1 - wpos, co = row & (RBF_C - 1);
    const int* th = which ? P.dh2 : P.dh1;
    const int* tw = which ? P.dw2 : P.dw1;
    int tap = -1;
    for (int t = 0; t < 9; ++t)
      if (th[t] == dh && tw[t] == dwi) tap = t;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (tap >= 0) v = *reinterpret_cast<const uint4*>((which ? P.w2 : P.w1) + ((size_t)tap * RBF_C + co) * RBF_C + j * 8);
    st_shared_v4((which ? sW2 : sW1) + (uint32_t)row * RBF_PIX + (uint32_t)((j ^ ((row >> 1) & 3)) << 4), v);
  }
  for (uint32_t o = threadIdx.x * 16u; o < (uint32_t)(XS + US) * SLOT; o += blockDim.x * 16u)
    st_shared_v4(sX + o, make_uint4(0u, 0u, 0u, 0u));
  if (threadIdx.x == 0) {
    for (int s = 0; s < XS; ++s) { mbar_init(xfull0 + 8u * s, 1); mbar_init(xempty0 + 8u * s, 1); }
    for (int s = 0; s < US; ++s) { mbar_init(ufull0 + 8u * s, 1); mbar_init(uempty0 + 8u * s, 1); }
    for (int s = 0; s < R; ++s) {
      mbar_init(t1done0 + 8u * s, 1); mbar_init(t1free0 + 8u * s, RBF_GROUP_WARPS * MT);
      mbar_init(t2done0 + 8u * s, 1); mbar_init(t2free0 + 8u * s, RBF_GROUP_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&tmX);
    if (!VJP) prefetch_tmap(&tmAct);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_async_smem();  // B operands and zeroed rings -> async proxy
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_holder, 0);
  if (warp >= 2 && warp < 18) {  // every ring block starts (and is returned by the epilogue) zeroed
    const uint32_t ta = tmem_base + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(((warp - 2) >> 2) * 128);
#pragma unroll
    for (int c = 0; c < 128; c += 8) tmem_zero8(ta + (uint32_t)c);
    tmem_st_wait();
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  // this CTA's rows of the live row sequence
  int nimg = P.N;
  if (P.act_list) nimg = ld_volatile_s32(P.n_act);
  const long long Q = (long long)nimg * P.H;
  const int q0 = (int)(Q * blockIdx.x / gridDim.x), q1 = (int)(Q * (blockIdx.x + 1) / gridDim.x);

  if (warp == 0) {
    // ---------------- producer: x rows h0-2 .. h1+1 of each run (run offsets 0 .. nu+1)
    uint32_t xc = 0;
    int q = q0;
    RbfRun run;
    while (rbf_next_run(P, q, q1, run)) {
      const int nx = run.h1 - run.h0 + 4;
      for (int k = 0; k < nx; ++k, ++xc) {
        const int s = (int)(xc % XS);
        mbar_wait_sleep(xempty0 + 8u * s, ((xc / XS) & 1u) ^ 1u);
        if (elect_one()) {
          mbar_expect_tx(xfull0 + 8u * s, (uint32_t)W * RBF_PIX);
          tma_load_4d(sX + (uint32_t)s * SLOT + 1024u, &tmX, xfull0 + 8u * s, 0, 0, run.h0 - 2 + k, run.n);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer
    const uint64_t dW1 = make_sdesc(sW1, 512u, 4u), dW2 = make_sdesc(sW2, 512u, 4u);
    uint32_t xc = 0, uc = 0, oc = 0;  // ring counters (input rows, intermediate rows, output rows)
    int q = q0;
    RbfRun run;
    // An input row (payload address) contributes to ring rows g_lo .. g_hi (global counters, <= 3,
    // window positions w_lo ..): 3 dw x 2 K steps, each one MMA -- N = 96 at the window's first
    // block, or for a full window that wraps N = 128 over the whole ring with the rotated B (the
    // clipped windows at run ends that wrap are split in two).
    // Descriptors are built once per window and stepped by constants: the single issuing thread's
    // instruction stream between MMAs is what bounds this loop otherwise (~150 clk per MMA with
    // per-MMA descriptor arithmetic vs 56 clk for the N = 96 MMA itself, tools/mma_rate_probe.cu).
    const uint32_t idesc32 = make_idesc_bf16(32);
    auto mma_window = [&](uint32_t stage_col, uint32_t payload, uint64_t dWb, uint32_t g_lo, uint32_t g_hi, int w_lo) {
      uint32_t b_lo = g_lo % R;
      const uint32_t n = g_hi - g_lo + 1;
      uint32_t n1 = min(n, (uint32_t)R - b_lo), n2 = n - n1;  // blocks before / after the wrap
      uint32_t bstart = (uint32_t)w_lo;                       // first B block of the window
      if (n == 3 && n2 != 0) {  // full window that wraps: N = 128 over blocks 0..3, B rotated
        bstart = b_lo == 2 ? 2u : 1u;
        b_lo = 0;
        n1 = 4;
        n2 = 0;
      }
      const uint32_t id1 = idesc32 + ((n1 - 1u) << 19), id2 = idesc32 + ((n2 - 1u) << 19);  // N >> 3 = 4 n
      const uint64_t b1 = dWb + (uint64_t)((bstart * RBF_WTAP) >> 4), b2 = b1 + (uint64_t)((n1 * RBF_WTAP) >> 4);
      const uint64_t a0 = make_sdesc(payload - RBF_PIX, 512u, 4u);  // dw = -1 window of M tile 0
      // the hot path (n2 == 0) is a straight run of MMAs: a branch between two tcgen05.mma
      // instructions costs far more issue time than the MMA's own ~60 clk
      if (RBF_NO_MMA) return;
      if (n2 == 0) {
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
          const uint32_t d1 = tmem_base + stage_col + (uint32_t)(mt * R * RBF_C) + b_lo * RBF_C;
          const uint64_t am = a0 + (uint64_t)(mt * 128 * (int)RBF_PIX / 16);
#pragma unroll
          for (int dwi = 0; dwi < 3; ++dwi)
#pragma unroll
            for (int k = 0; k < 2; ++k)
              mma_bf16_elect(d1, am + (uint64_t)(dwi * (int)RBF_PIX / 16 + 2 * k),
                             b1 + (uint64_t)(dwi * (int)RBF_WGROUP / 16 + 2 * k), id1, 1u);
        }
      } else {
#pragma unroll 1
        for (int mt = 0; mt < MT; ++mt) {
          const uint32_t d1 = tmem_base + stage_col + (uint32_t)(mt * R * RBF_C) + b_lo * RBF_C;
          const uint32_t d2 = tmem_base + stage_col + (uint32_t)(mt * R * RBF_C);
          const uint64_t am = a0 + (uint64_t)(mt * 128 * (int)RBF_PIX / 16);
#pragma unroll
          for (int dwi = 0; dwi < 3; ++dwi)
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const uint64_t ad = am + (uint64_t)(dwi * (int)RBF_PIX / 16 + 2 * k);
              const uint64_t boff = (uint64_t)(dwi * (int)RBF_WGROUP / 16 + 2 * k);
              mma_bf16_elect(d1, ad, b1 + boff, id1, 1u);
              mma_bf16_elect(d2, ad, b2 + boff, id2, 1u);
            }
        }
      }
    };
    while (rbf_next_run(P, q, q1, run)) {
      const int nu = run.h1 - run.h0 + 2, no = run.h1 - run.h0;
      const uint32_t xb = xc, ub = uc, ob = oc;
      // S1(k): input row k (image row h0-2+k) -> intermediate rows iu = k-2 .. k (image row h0-1+iu)
      auto s1 = [&](int k) {
        if (lane == 0) RBF_EV(2, k);
        const uint32_t c = xb + (uint32_t)k;
        mbar_wait(xfull0 + 8u * (c % XS), (c / XS) & 1u);
        const int lo = max(0, k - 2), hi = min(k, nu - 1);
        if (k < nu) {  // first contribution to intermediate row k: its block must be back (zeroed)
          const uint32_t g = ub + (uint32_t)k;
          mbar_wait(t1free0 + 8u * (g % R), ((g / R) & 1u) ^ 1u);
          // a wrapping full window adds +0 to the fourth block: wait until the epilogue has drained it
          if (k >= 2 && ((g - 2u) % R) >= 2u) mbar_wait(t1free0 + 8u * ((g + 1u) % R), (((g + 1u) / R) & 1u) ^ 1u);
        }
        tc_fence_after();
        if (lane == 0) RBF_EV(4, k);
        mma_window(0u, sX + (c % XS) * SLOT + 1024u, dW1, ub + (uint32_t)lo, ub + (uint32_t)hi, lo - (k - 2));
        mma_commit_elect(xempty0 + 8u * (c % XS));  // input row k has no other reader
        if (k >= 2) mma_commit_elect(t1done0 + 8u * ((ub + (uint32_t)(k - 2)) % R));
      };
      // S2(j): intermediate row j -> output rows io = j-2 .. j (image row h0+io)
      auto s2 = [&](int j) {
        if (lane == 0) RBF_EV(5, j);
        const uint32_t c = ub + (uint32_t)j;
        mbar_wait(ufull0 + 8u * (c % US), (c / US) & 1u);
        const int lo = max(0, j - 2), hi = min(j, no - 1);
        if (j < no) {
          const uint32_t g = ob + (uint32_t)j;
          mbar_wait(t2free0 + 8u * (g % R), ((g / R) & 1u) ^ 1u);
          if (j >= 2 && ((g - 2u) % R) >= 2u) mbar_wait(t2free0 + 8u * ((g + 1u) % R), (((g + 1u) / R) & 1u) ^ 1u);
        }
        tc_fence_after();
        if (lane == 0) RBF_EV(7, j);
        if (lo <= hi)
          mma_window((uint32_t)(MT * R * RBF_C), sU + (c % US) * SLOT + 1024u, dW2, ob + (uint32_t)lo, ob + (uint32_t)hi,
                     lo - (j - 2));
        mma_commit_elect(uempty0 + 8u * (c % US));
        if (j >= 2 && j - 2 < no) mma_commit_elect(t2done0 + 8u * ((ob + (uint32_t)(j - 2)) % R));
      };
      for (int k = 0; k <= nu + 1; ++k) {
        s1(k);
        if (k >= 3) s2(k - 3);
      }
      s2(nu - 1);
      xc += (uint32_t)(nu + 2);
      uc += (uint32_t)nu;
      oc += (uint32_t)no;
    }
  } else {
    // ---------------- epilogue: two independent warp groups, so a slow stage-2 row never holds up
    // the stage-1 epilogue the MMA warp is waiting on (and vice versa). Group 0 (warps 2 ..
    // 1 + 8 MT): E1, one M tile per warp (tile = (warp - 2) / 8), group 1 (the last 8 warps): E2,
    // every tile; in a group, warp -> (TMEM lane quadrant, 16-channel half).
    constexpr int E1W = RBF_GROUP_WARPS * MT;
    const int grp = warp - 2 < E1W ? 0 : 1;
    const int gw = grp == 0 ? (warp - 2) % RBF_GROUP_WARPS : warp - 2 - E1W;
    const int e1_mt = grp == 0 ? (warp - 2) / RBF_GROUP_WARPS : 0;
    const int quad = warp & 3, half = gw >> 2;
    const int c0 = half * 16;  // this warp's 16 channels = 16-byte chunks 2 half, 2 half + 1
    const bool leader = warp == 2 && lane == 0;
    uint32_t uc = 0, oc = 0;
    int q = q0;
    RbfRun run;
    const uint32_t tq = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)c0;
    // read this warp's 16 columns of ring block `blk` of a stage for M tiles [m0, m0 + NM) and zero them
    auto drain = [&](uint32_t stage_col, uint32_t blk, int m0, auto nm_tag, uint32_t (&v)[decltype(nm_tag)::value][16]) {
      constexpr int NM = decltype(nm_tag)::value;
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        uint32_t a[8], b[8];
        tmem_ld8_nw(tq + stage_col + (uint32_t)((m0 + i) * R * RBF_C) + blk * RBF_C, a);
        tmem_ld8_nw(tq + stage_col + (uint32_t)((m0 + i) * R * RBF_C) + blk * RBF_C + 8u, b);
        tmem_wait();
#pragma unroll
        for (int e = 0; e < 8; ++e) { v[i][e] = a[e]; v[i][8 + e] = b[e]; }
      }
#pragma unroll
      for (int i = 0; i < NM; ++i) {
        tmem_zero8(tq + stage_col + (uint32_t)((m0 + i) * R * RBF_C) + blk * RBF_C);
        tmem_zero8(tq + stage_col + (uint32_t)((m0 + i) * R * RBF_C) + blk * RBF_C + 8u);
      }
    };
    auto give_back = [&](uint32_t free_bar) {  // after drain: the zeros have landed, block is free
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(free_bar);
    };
    // 16 channels of pixel p of a row: two 16-byte chunks
    auto gload2 = [&](const __nv_bfloat16* base, size_t pix, uint4 (&o)[2]) {
      const uint4* g = reinterpret_cast<const uint4*>(base + pix * RBF_C + c0);
      o[0] = __ldg(g);
      o[1] = __ldg(g + 1);
    };
    // VJP: the saved-activation chunks of the next stage-1 row (this warp's tile), prefetched one row ahead
    uint4 av[2];
    int av_row = -1;  // image row (in image av_n) av holds, -1: none
    int av_n = -1;
    const int p1 = 128 * e1_mt + quad * 32 + lane;  // E1: this thread's pixel of the row
    auto load_a = [&](int n, int h) {
      gload2(P.act, ((size_t)n * P.H + h) * W + p1, av);
      av_n = n;
      av_row = h;
    };
    while (rbf_next_run(P, q, q1, run)) {
      const int nu = run.h1 - run.h0 + 2, no = run.h1 - run.h0;
      const uint32_t ub = uc, ob = oc;
      if (grp == 0) {
        // E1: intermediate row iu (image row h0-1+iu) -> u ring (+ forward: a to HBM)
        for (int iu = 0; iu < nu; ++iu) {
          const int h = run.h0 - 1 + iu;
          const bool inside = h >= 0 && h < P.H;
          const uint32_t g = ub + (uint32_t)iu;
          if (VJP && inside && (av_row != h || av_n != run.n)) load_a(run.n, h);
          if (leader) RBF_EV(8, iu);
          mbar_wait_sleep(uempty0 + 8u * (g % US), ((g / US) & 1u) ^ 1u);
          mbar_wait_sleep(t1done0 + 8u * (g % R), (g / R) & 1u);
          tc_fence_after();
          if (leader) RBF_EV(9, iu);
          if (RBF_NO_EPI) {
            rbf_epi_bar<MT>();
            if (leader) mbar_arrive(ufull0 + 8u * (g % US));
            __syncwarp();
            if (lane == 0) mbar_arrive(t1free0 + 8u * (g % R));
            continue;
          }
          uint32_t d[1][16];
          drain(0u, g % R, e1_mt, std::integral_constant<int, 1>{}, d);
          const uint32_t upl = sU + (g % US) * SLOT + 1024u;
          uint4 w[2];
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            w[jj] = make_uint4(0u, 0u, 0u, 0u);
            if (inside) {
              float v[8];
              if (VJP) {  // q = (B^T g) . sp'(a)
                const __nv_bfloat162* a2 = reinterpret_cast<const __nv_bfloat162*>(&av[jj]);
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  const float2 f = __bfloat1622float2(a2[e]);
                  v[2 * e] = __uint_as_float(d[0][8 * jj + 2 * e]) * dsoftplus_from_act_fast(f.x);
                  v[2 * e + 1] = __uint_as_float(d[0][8 * jj + 2 * e + 1]) * dsoftplus_from_act_fast(f.y);
                }
              } else {  // a = sp(A t)
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                  const float t = __uint_as_float(d[0][8 * jj + e]);
                  v[e] = (e & 1) ? softplus_poly_log(t) : softplus_fast(t);
                }
              }
              __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&w[jj]);
#pragma unroll
              for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
            }
            st_shared_v4(rbf_chunk(upl, p1, 2 * half + jj), w[jj]);
          }
          fence_async_smem();  // u row -> async proxy (stage-2 MMAs, the act store)
          // the u slot written next row (US - 1 rows after this one) must have been read by its
          // act store, issued US - 1 rows ago: at most US - 2 stores may still be reading
          if (!VJP && leader) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(US - 2) : "memory");
          rbf_epi_bar<MT>();
          if (leader) { mbar_arrive(ufull0 + 8u * (g % US)); RBF_EV(10, iu); }
          if (!VJP && leader && inside) {  // the saved activation a, straight from the u row
            tma_store_4d(upl, &tmAct, 0, 0, h, run.n);
            bulk_commit();
          }
          give_back(t1free0 + 8u * (g % R));
          if (VJP && iu + 1 < nu && h + 1 < P.H) load_a(run.n, h + 1);  // latency hidden by the next waits
          // VJP: the saved-activation row three rows ahead is pulled into L2 by one bulk prefetch, so
          // the per-thread loads above (one row ahead) hit L2 instead of waiting on HBM
          if (VJP && leader && iu + 3 < nu && h + 3 < P.H)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(P.act + ((size_t)run.n * P.H + h + 3) * W * RBF_C),
                         "r"((uint32_t)(W * RBF_PIX))
                         : "memory");
        }
      } else {
        // E2: output row io (image row h0+io) = residual + conv 2
        for (int io = 0; io < no; ++io) {
          const uint32_t g = ob + (uint32_t)io;
          const size_t rowoff = ((size_t)run.n * P.H + run.h0 + io) * W;
          uint4 rv[MT][2];  // the residual (block input row h0+io), loaded from L2 before the wait
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) gload2(P.x, rowoff + 128 * mt + quad * 32 + lane, rv[mt]);
          if (gw == 0 && lane == 0) RBF_EV(11, io);
          mbar_wait_sleep(t2done0 + 8u * (g % R), (g / R) & 1u);
          tc_fence_after();
          if (gw == 0 && lane == 0) RBF_EV(12, io);
          if (RBF_NO_EPI) {
            __syncwarp();
            if (lane == 0) mbar_arrive(t2free0 + 8u * (g % R));
            continue;
          }
          uint32_t d[MT][16];
          drain((uint32_t)(MT * R * RBF_C), g % R, 0, std::integral_constant<int, MT>{}, d);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) {
            uint4 w[2];
#pragma unroll
            for (int jj = 0; jj < 2; ++jj) {
              const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&rv[mt][jj]);
              __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&w[jj]);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(r2[e]);
                h2[e] = __floats2bfloat162_rn(__uint_as_float(d[mt][8 * jj + 2 * e]) + f.x,
                                              __uint_as_float(d[mt][8 * jj + 2 * e + 1]) + f.y);
              }
            }
            uint4* o = reinterpret_cast<uint4*>(P.out + (rowoff + 128 * mt + quad * 32 + lane) * RBF_C + c0);
            o[0] = w[0];
            o[1] = w[1];
          }
          give_back(t2free0 + 8u * (g % R));
          if (gw == 0 && lane == 0) RBF_EV(13, io);
        }
      }
      uc += (uint32_t)nu;
      oc += (uint32_t)no;
    }
  }
  if (!VJP && warp == 2 && lane == 0) bulk_wait0();  // the act stores are complete
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(512) : "memory");
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn4)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn4 rbf_encode() {
  static EncodeTiledFn4 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn4>(p);
  }
  return fn;
}

struct RbfPlan {
  CUtensorMap tmX;
  CUtensorMap tmAct;  // forward: the saved activation (same layout as x)
  RbfParams P;
  const int* list_ptr;
  bool vjp;
  int grid;
  size_t smem;
};

bool rbf_supported(int W, int C) { return C == RBF_C && (W == 128 || W == 256); }

static CUresult rbf_map(EncodeTiledFn4 enc, CUtensorMap* m, const void* p, int N, int H, int W) {
  cuuint64_t dims[4] = {(cuuint64_t)RBF_C, (cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[3] = {(cuuint64_t)RBF_PIX, (cuuint64_t)RBF_PIX * W, (cuuint64_t)RBF_PIX * W * H};
  cuuint32_t box[4] = {(cuuint32_t)RBF_C, (cuuint32_t)W, 1u, 1u};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(p), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

RbfPlan* rbf_make_plan(bool vjp, int N, int H, int W, const int dh1[9], const int dw1[9], const int dh2[9],
                       const int dw2[9], const __nv_bfloat16* w1, const __nv_bfloat16* w2, const void* x, void* out,
                       void* act, int num_sms, char* err, size_t errlen) {
  if (!rbf_supported(W, RBF_C)) { snprintf(err, errlen, "fused residual block: unsupported width"); return nullptr; }
  EncodeTiledFn4 enc = rbf_encode();
  if (!enc) { snprintf(err, errlen, "cuTensorMapEncodeTiled unavailable"); return nullptr; }
  RbfPlan* p = new RbfPlan();
  memset(p, 0, sizeof(RbfPlan));
  p->vjp = vjp;
  RbfParams& P = p->P;
  P.N = N; P.H = H; P.W = W;
  for (int t = 0; t < 9; ++t) { P.dh1[t] = dh1[t]; P.dw1[t] = dw1[t]; P.dh2[t] = dh2[t]; P.dw2[t] = dw2[t]; }
  P.w1 = w1; P.w2 = w2;
  P.x = static_cast<const __nv_bfloat16*>(x);
  P.out = static_cast<__nv_bfloat16*>(out);
  P.act = static_cast<__nv_bfloat16*>(act);
  CUresult r = rbf_map(enc, &p->tmX, x, N, H, W);
  if (r == CUDA_SUCCESS && !vjp) r = rbf_map(enc, &p->tmAct, act, N, H, W);
  if (r != CUDA_SUCCESS) { snprintf(err, errlen, "fused residual block: tensor map encode failed (%d)", (int)r); delete p; return nullptr; }
  p->smem = W == 128 ? RbfCfg<1>::smem() : RbfCfg<2>::smem();
  const long long rows = (long long)N * H;
  p->grid = (int)(rows < num_sms ? rows : num_sms);
  return p;
}

void rbf_set_active(RbfPlan* p, const int* act_list, const int* n_act) {
  p->list_ptr = act_list;
  p->P.n_act = n_act;
  p->P.act_list = nullptr;
}
void rbf_enable_skip(RbfPlan* p, bool on) { p->P.act_list = on ? p->list_ptr : nullptr; }
void rbf_free_plan(RbfPlan* p) { delete p; }

void rbf_launch(const RbfPlan* p, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p->grid);
  cfg.blockDim = dim3(p->P.W == 128 ? rbf_threads<1>() : rbf_threads<2>());
  cfg.dynamicSmemBytes = p->smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const bool narrow = p->P.W == 128;
  if (p->vjp) {
    if (narrow) cudaLaunchKernelEx(&cfg, rbf_kernel<1, true>, p->tmX, p->tmX, p->P);
    else cudaLaunchKernelEx(&cfg, rbf_kernel<2, true>, p->tmX, p->tmX, p->P);
  } else {
    if (narrow) cudaLaunchKernelEx(&cfg, rbf_kernel<1, false>, p->tmX, p->tmAct, p->P);
    else cudaLaunchKernelEx(&cfg, rbf_kernel<2, false>, p->tmX, p->tmAct, p->P);
  }
}

void init_attrs_rbf() {
  set_max_dyn_smem(rbf_kernel<1, false>);
  set_max_dyn_smem(rbf_kernel<1, true>);
  set_max_dyn_smem(rbf_kernel<2, false>);
  set_max_dyn_smem(rbf_kernel<2, true>);
}

}  // namespace ideq
