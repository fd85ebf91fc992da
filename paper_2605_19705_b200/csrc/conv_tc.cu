// tcgen05 / TMEM / TMA implicit-GEMM convolution for sm_100a (bf16 operands, fp32
// accumulation in tensor memory) with the i-DEQ epilogues fused:
//   forward  RB conv A : a = softplus(W * t)         (saved for the VJP)
//   forward  RB conv B : t' = t + W * a
//   adjoint  conv B^T  : q = (W~ * g) . sp'(a)        (sp' recomputed from saved a)
//   adjoint  conv A^T  : g' = g + W~ * q
//   2x2 stride-2 down / transposed up and their adjoints (patch / scatter geometry).
//
// GEMM view (ConvGeom in common.cuh): M = 128 output pixels of an R x Wt tile,
// N = GEMM columns (output channels, or 4 x channels for the scatter layers),
// K = taps x input channels, walked in K-blocks of KC = 32/64 channels of one tap.
//
// Warp roles (192 threads, persistent over tiles):
//   warp 0      : TMA producer -- one 5-D box (KC ch x Wt x 1 x R x 1) of the input per
//                 K-block (out-of-range rows/cols are zero-filled by TMA = conv padding)
//                 and one 3-D box of the pre-arranged weights [kb][ncols][KC].
//   warp 1      : TMEM allocator + single-thread tcgen05.mma issuer (M=128, N=BN, K=16),
//                 tcgen05.commit frees smem stages and publishes accumulators.
//   warps 2..5  : epilogue -- tcgen05.ld 32 lanes x 32 columns, fused activation /
//                 residual / sp' multiply, bf16 pack, 16-byte global stores.
// TMEM holds two BN-column accumulators so the epilogue of tile i overlaps the MMAs
// of tile i+1. Shared-memory stages form an mbarrier ring (full/empty).
#include <cuda.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace ideq {

// Bisection switches for timing studies only (tools/build_variant.sh, tools/run_gpu_s2j.sh ->
// profiles/r2c_conv_bisect.txt; results are NOT correct with any of them on, the product build
// leaves them 0): TCX_NO_EPI -- the epilogue only hands the accumulator back (no TMEM loads, math
// or stores); TCX_NO_B -- streamed weights are neither loaded nor waited for; TCX_NO_A -- the input
// boxes are not loaded (the producer arrives without data).
#ifndef TCX_NO_EPI
#define TCX_NO_EPI 0
#endif
#ifndef TCX_NO_B
#define TCX_NO_B 0
#endif
#ifndef TCX_NO_A
#define TCX_NO_A 0
#endif

// ------------------------------------------------------------------ PTX helpers
// ------------------------------------------------------------------ kernel
struct TcParams {
  ConvGeom g;
  int BN, n_tiles, m_tiles, stages;
  uint32_t a_bytes, b_bytes, tmem_cols;
  uint32_t epi_box_bytes;  // one epilogue box: 128 rows x BOXC columns (bf16)
  uint32_t epi_tx_bytes;   // TMA bytes of one aux tile (R*Wt rows x BN columns)
  uint32_t halo_stage;     // HALO: bytes of one (Wt+2) x (R+2) x KC halo buffer (1 KB aligned)
  int stagesB;             // MODE 2: depth of the weight ring
  int nacc;                // TMEM accumulator stages (2..8)
  int nepi;                // epilogue staging buffers (<= nacc): tile k uses accumulator k % nacc and
                           // buffer k % nepi
  int nsplit;              // 3xTF32: partial accumulators per tile (summed in fp32 by the epilogue)
  // EPI_IMG: the first img_c GEMM columns are an image (tail / head adjoint); written as fp32
  // NCHW planes [N][img_c][OH][OW] plus img_alpha * img_aux (same layout, may be null)
  float* img_out;
  const float* img_aux;
  float img_alpha;
  int img_c;
  FastDiv fd_ntiles, fd_perimg, fd_tw;  // tile index -> (m tile, n tile), (image, row tile, col tile)
  int slab_mode;                        // 1: each TMEM lane quadrant stores its own 32-row slab
  // live-tile list (tol > 0 per-image solves): the solver keeps a compacted list of its active
  // images (act_list[0 .. *n_act)); every warp role walks the tiles of those images only, in the
  // same order, so work stays balanced over the CTAs when images freeze (null: every tile)
  const int* act_list;
  const int* n_act;
  FastDiv fd_tpi;   // tiles per image (M tiles x N tiles)
  int tpi;
};

// k-th live tile -> raw tile index (identity without a live list). The list lives in global
// memory (written by the previous iteration's bookkeeping kernel) and is read through the
// read-only path; every role computes the same sequence.
__device__ __forceinline__ int live_tile(const TcParams& P, int L) {
  if (!P.act_list) return L;
  const int q = (int)P.fd_tpi.div((uint32_t)L);
  return __ldg(P.act_list + q) * P.tpi + (L - q * P.tpi);
}

// tile t -> (image, output row h0, output col w0, n tile)
struct TileIdx { int img, h0, w0, nt; };
__device__ __forceinline__ TileIdx tile_index(const TcParams& P, int t) {
  TileIdx r;
  const int mt = (int)P.fd_ntiles.div((uint32_t)t);
  r.nt = t - mt * P.n_tiles;
  r.img = (int)P.fd_perimg.div((uint32_t)mt);
  const int rem = mt - r.img * (P.g.tiles_h * P.g.tiles_w);
  const int th = (int)P.fd_tw.div((uint32_t)rem);
  r.h0 = th * P.g.R;
  r.w0 = (rem - th * P.g.tiles_w) * P.g.Wt;
  return r;
}

constexpr int TC_THREADS = 352;     // warp 0 TMA operands, warp 1 MMA, warps 2..9 epilogue, warp 10 TMA aux
constexpr int TC_THREADS_X3 = 480;  // 3xTF32: + warps 11..14 split every staged fp32 A tile into tf32 hi / lo

// MODE (3x3 convs): 0 = plain implicit GEMM, one TMA box of the shifted input per (tap, chunk).
// 1 and 2 = HALO: one TMA box of (Wt+2) x (R+2) input pixels per channel chunk feeds all 9 taps
// through shifted UMMA descriptors. The M = 128 rows of a tile are either one image row of 128
// pixels (R = 1) or 16 rows x 8 pixels (Wt = 8), the two shapes whose 8-row core groups sit at a
// uniform stride inside the halo box (8 or 10 pixel rows = the descriptor's SBO), so the input
// crosses L2 ~1.4x (2D) / ~3x (1-row) instead of 9x. MODE 1 keeps the layer's weights resident
// in shared memory for the CTA's lifetime; MODE 2 streams them per (chunk, tap) through a second
// ring (layers whose weights do not fit).
//
// KB = bytes of one K-block row (one pixel's channel chunk): 64 (SW64) or 128 (SW128); one MMA
// consumes 32 bytes of K (16 bf16 / 8 tf32). BOXB = bytes of one epilogue-box row (64 or 128).
//
// X3 (the fp32 parity mode, 3xTF32): operands are fp32 in HBM. The weights arrive pre-split into
// tf32 hi / lo tensors (tmB, tmBlo); every staged fp32 A tile is split in shared memory by four
// converter warps (hi in place, lo beside it) before the MMA warp may read it, and every K step
// issues A_hi*B_hi + A_lo*B_hi + A_hi*B_lo (kind::tf32) into the fp32 TMEM accumulator
// (the A_lo*B_lo term is below fp32 rounding). The epilogue keeps fp32 and the exact fp32
// softplus / sp'. Reference: the network of Eq. 2 and its VJP.
template <int KB, int EPI, int BOXB, int MODE, bool X3>
__global__ void __launch_bounds__(X3 ? TC_THREADS_X3 : TC_THREADS, X3 ? 1 : 2)
    conv_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmOut, const __grid_constant__ CUtensorMap tmAux,
                   const __grid_constant__ CUtensorMap tmSlab, const __grid_constant__ CUtensorMap tmBlo,
                   const __grid_constant__ TcParams P) {
  constexpr bool HAS_AUX = (EPI == EPI_RESADD || EPI == EPI_SIGMUL);
  constexpr int ES = X3 ? 4 : 2;           // element bytes (fp32 / bf16)
  constexpr int BOXC = BOXB / ES;          // columns per epilogue box
  constexpr int NBUF = X3 ? 2 : 1;         // operand buffers per stage (hi, lo)
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
  const int S = P.stages;
  const int BN = P.BN;
  const uint32_t a_stage = 128u * KB;
  constexpr bool STREAMB = MODE == 2;
  const uint32_t b_stage = (uint32_t)BN * KB;             // one weight box (hi or lo)
  const uint32_t bslot = b_stage * NBUF;                  // one ring slot: hi (+ lo)
  const uint32_t epi_stage = (uint32_t)BN * 128u * ES;    // BN/BOXC boxes of 128 x BOXC
  const ConvGeom& g = P.g;
  const int nkb = g.ntaps * g.nchunk;
  constexpr bool HALO = MODE != 0;
  const int SB = STREAMB ? P.stagesB : 0;
  const uint32_t op_a = HALO ? P.halo_stage : a_stage;    // one A buffer (hi or lo)
  // MODE 0: [A hi S][A lo S][B slots S][epi]; MODE 1: [W hi nkb][W lo nkb][halo hi S][halo lo S][epi];
  // MODE 2: [halo hi S][halo lo S][B ring slots SB][epi]      (lo buffers in 3xTF32 only)
  const uint32_t sW = base;
  const uint32_t sA = (MODE == 1) ? sW + (uint32_t)nkb * bslot : base;
  const uint32_t sAlo = sA + S * op_a;
  const uint32_t sB = sA + S * op_a * NBUF;
  const uint32_t sE = (MODE == 1) ? sB : sB + (STREAMB ? SB : S) * bslot;
  const int NA = P.nacc;  // TMEM accumulator stages
  const int NE = P.nepi;  // epilogue buffers
  const uint32_t sBar = sE + (uint32_t)NE * epi_stage;
  uint64_t* bars = reinterpret_cast<uint64_t*>(gbase + (sBar - base));
  // barriers: full[S], empty[S], tfull[NA], tempty[NA], auxfull[NA], epifree[NA], wfull, fullB[SB],
  // emptyB[SB], split[S] (3xTF32: the A tile of stage s is split)
  const int NSPL = X3 ? S : 0;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * S + 4 * NA + 1 + 2 * SB + NSPL);
  const uint32_t full0 = sBar, empty0 = sBar + 8u * S;
  const uint32_t tfull0 = sBar + 16u * S, tempty0 = tfull0 + 8u * NA, auxfull0 = tempty0 + 8u * NA,
                 epifree0 = auxfull0 + 8u * NA;
  const uint32_t wfull = epifree0 + 8u * NA;
  const uint32_t fullB0 = wfull + 8u, emptyB0 = fullB0 + 8u * SB;
  const uint32_t split0 = emptyB0 + 8u * SB;
  // the MMA warp waits for the split tile (3xTF32) or the landed tile
  const uint32_t ready0 = X3 ? split0 : full0;

  // warp index broadcast from lane 0 so the compiler knows it is warp-uniform (uniform datapath)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  // Programmatic dependent launch: the next layer may be scheduled now; its CTAs run their
  // prologue as SMs free up and wait (griddepcontrol.wait) for this grid before touching data.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (threadIdx.x == 0) {
    mbar_init(wfull, 1);
    if (MODE == 1) {  // resident weights (constant since create): loaded before the wait
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(wfull, (uint32_t)nkb * P.b_bytes * NBUF);
      for (int kb = 0; kb < nkb; ++kb) tma_load_3d(sW + kb * b_stage, &tmB, wfull, 0, 0, kb);
      if (X3)
        for (int kb = 0; kb < nkb; ++kb) tma_load_3d(sW + (nkb + kb) * b_stage, &tmBlo, wfull, 0, 0, kb);
    }
    for (int s = 0; s < S; ++s) { mbar_init(full0 + 8u * s, 1); mbar_init(empty0 + 8u * s, 1); }
    for (int s = 0; s < SB; ++s) { mbar_init(fullB0 + 8u * s, 1); mbar_init(emptyB0 + 8u * s, 1); }
    for (int s = 0; s < NSPL; ++s) mbar_init(split0 + 8u * s, 4);  // one arrival per converter warp
    for (int a = 0; a < NA; ++a) {
      mbar_init(tfull0 + 8u * a, 1);
      mbar_init(tempty0 + 8u * a, 8);   // one arrival per epilogue warp
      mbar_init(auxfull0 + 8u * a, 1);
      mbar_init(epifree0 + 8u * a, 4);  // one arrival per TMEM lane quadrant
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    prefetch_tmap(&tmOut);
    prefetch_tmap(&tmSlab);
    if (HAS_AUX) prefetch_tmap(&tmAux);
    if (X3) prefetch_tmap(&tmBlo);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // everything below reads what earlier kernels wrote: wait for them (no-op without PDL)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_holder, 0);  // uniform, not a per-thread load

  const int total = P.m_tiles * P.n_tiles;
  const int t0 = (int)blockIdx.x;
  const int tstep = (int)gridDim.x;
  const int nbox = BN / BOXC;
  // tiles this launch walks: all of them, or the live list's (read after griddepcontrol.wait)
  int tot_it = total;
  if (P.act_list) tot_it = ld_volatile_s32(P.n_act) * P.tpi;
  const int nload = HALO ? g.nchunk : nkb;  // A stages per tile

  if (warp == 0) {
    // ---------------- TMA producer: the whole warp walks the loop (warp-uniform state stays in
    // uniform registers); one elected lane arms the barriers and issues the copies
    int s = 0, sb = 0;
    uint32_t ph = 0, phb = 0;
    for (int L = t0; L < tot_it; L += tstep) {
      const TileIdx ti = tile_index(P, live_tile(P, L));
      const int img = ti.img, h0 = ti.h0, w0 = ti.w0, nt = ti.nt;
      for (int kb = 0; kb < nload; ++kb) {
        mbar_wait(empty0 + 8u * s, ph ^ 1u);
        if (elect_one()) {
          if (HALO) {
            if (TCX_NO_A) {
              mbar_arrive(full0 + 8u * s);
            } else {
              mbar_expect_tx(full0 + 8u * s, P.a_bytes);
              tma_load_5d(sA + s * op_a, &tmA, full0 + 8u * s, kb * (KB / ES), w0 - 1, 0, h0 - 1, img);
            }
            if (MODE == 2 && !TCX_NO_B) {  // this chunk's 9 weight boxes (hi, lo) through the B ring
              for (int tap = 0; tap < 9; ++tap) {
                mbar_wait(emptyB0 + 8u * sb, phb ^ 1u);
                mbar_expect_tx(fullB0 + 8u * sb, P.b_bytes * NBUF);
                tma_load_3d(sB + sb * bslot, &tmB, fullB0 + 8u * sb, 0, nt * BN, tap * g.nchunk + kb);
                if (X3) tma_load_3d(sB + sb * bslot + b_stage, &tmBlo, fullB0 + 8u * sb, 0, nt * BN, tap * g.nchunk + kb);
                if (++sb == SB) { sb = 0; phb ^= 1u; }
              }
            }
          } else {
            const int tap = kb / g.nchunk, chunk = kb - tap * g.nchunk;
            mbar_expect_tx(full0 + 8u * s, P.a_bytes + P.b_bytes * NBUF);
            tma_load_5d(sA + s * a_stage, &tmA, full0 + 8u * s, chunk * (KB / ES), w0 + g.dw[tap], g.dp[tap],
                        h0 + g.dh[tap], img);
            tma_load_3d(sB + s * bslot, &tmB, full0 + 8u * s, 0, nt * BN, kb);
            if (X3) tma_load_3d(sB + s * bslot + b_stage, &tmBlo, full0 + 8u * s, 0, nt * BN, kb);
          }
        }
        __syncwarp();
        if (++s == S) { s = 0; ph ^= 1u; }
      }
    }
  } else if (X3 && warp >= 11) {
    // ---------------- 3xTF32 converter warps 11..14: split each landed fp32 A tile (the whole
    // staged box, element-wise, so the swizzle is irrelevant) into hi (in place) and lo
    const int ct = threadIdx.x - 11 * 32;  // 0..127
    int s = 0;
    uint32_t ph = 0;
    const uint32_t nchunks = P.a_bytes >> 4;
    for (int L = t0; L < tot_it; L += tstep) {
      for (int kb = 0; kb < nload; ++kb) {
        mbar_wait(full0 + 8u * s, ph);
        const uint32_t hi0 = sA + s * op_a, lo0 = sAlo + s * op_a;
        for (uint32_t c = ct; c < nchunks; c += 128) {
          const uint4 u = ld_shared_v4(hi0 + (c << 4));
          float h[4], l[4];
          split_tf32(__uint_as_float(u.x), h[0], l[0]);
          split_tf32(__uint_as_float(u.y), h[1], l[1]);
          split_tf32(__uint_as_float(u.z), h[2], l[2]);
          split_tf32(__uint_as_float(u.w), h[3], l[3]);
          st_shared_v4(hi0 + (c << 4), make_uint4(__float_as_uint(h[0]), __float_as_uint(h[1]), __float_as_uint(h[2]),
                                                  __float_as_uint(h[3])));
          st_shared_v4(lo0 + (c << 4), make_uint4(__float_as_uint(l[0]), __float_as_uint(l[1]), __float_as_uint(l[2]),
                                                  __float_as_uint(l[3])));
        }
        fence_async_smem();  // generic-proxy writes -> visible to the tensor core (async proxy)
        __syncwarp();
        if (lane == 0) mbar_arrive(split0 + 8u * s);
        if (++s == S) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 10) {
    // ---------------- aux producer: the epilogue's second operand (residual / saved activation)
    // goes into the tile's epilogue buffer as soon as that buffer's previous store has been read,
    // without ever stalling the operand producer behind the epilogue
    if (HAS_AUX) {
      int acc = 0;
      uint32_t aph = 0;
      for (int L = t0; L < tot_it; L += tstep) {
        const TileIdx ti = tile_index(P, live_tile(P, L));
        mbar_wait(epifree0 + 8u * acc, aph ^ 1u);
        if (elect_one()) {
          mbar_expect_tx(auxfull0 + 8u * acc, P.epi_tx_bytes);
          for (int b = 0; b < nbox; ++b) {
            const int col = ti.nt * BN + b * BOXC;
            tma_load_5d(sE + acc * epi_stage + b * P.epi_box_bytes, &tmAux, auxfull0 + 8u * acc, col % g.CB, ti.w0,
                        col / g.CB, ti.h0, ti.img);
          }
        }
        __syncwarp();
        if (++acc == NE) { acc = 0; aph ^= 1u; }  // (aux producer: epilogue buffers)
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the whole warp runs the loop with warp-uniform descriptors
    // (64-bit adds of byte offsets >> 4); one elected lane issues tcgen05.mma / commit. A
    // single-thread issue loop measured ~110 clk per MMA on B200 (tools/umma_bench.cu) against
    // a tensor floor of 16-128 clk; the uniform form reaches the floor for N >= 128.
    const uint32_t idesc = X3 ? make_idesc_tf32(BN) : make_idesc_bf16(BN);
    constexpr uint32_t layout = (KB == 128) ? 2u : 4u;   // SW128 / SW64
    constexpr uint32_t sbo = (KB == 128) ? 1024u : 512u; // 8 rows x row bytes
    // halo tiles: 8-row core groups of A are 8 pixels of one row (R = 1) or one 8-pixel row of a
    // 16 x 8 tile, i.e. (Wt + 2) pixel rows apart inside the halo box
    const uint32_t sboA = HALO ? (g.R == 1 ? sbo : (uint32_t)(g.Wt + 2) * KB) : sbo;
    const uint64_t dA0 = make_sdesc(sA, sboA, layout);
    const uint64_t dB0 = make_sdesc(MODE == 1 ? sW : sB, sbo, layout);
    const uint64_t loA = (uint64_t)((sAlo - sA) >> 4);                                   // A lo - A hi
    const uint64_t loB = (uint64_t)(((MODE == 1 ? (uint32_t)nkb * b_stage : b_stage)) >> 4);  // B lo - B hi
    int s = 0, sb = 0;
    uint32_t ph = 0, phb = 0;
    int acc = 0;
    uint32_t aph = 0;
    if (MODE == 1) mbar_wait(wfull, 0);
    auto mma_k = [&](uint32_t d_tmem, uint64_t ad, uint64_t bd, uint32_t first) {
#pragma unroll
      for (int k = 0; k < KB / 32; ++k) {
        if (X3) {
          mma_tf32_elect(d_tmem, ad + 2u * k, bd + 2u * k, idesc, (first | k) ? 1u : 0u);
          mma_tf32_elect(d_tmem, ad + loA + 2u * k, bd + 2u * k, idesc, 1u);
          mma_tf32_elect(d_tmem, ad + 2u * k, bd + loB + 2u * k, idesc, 1u);
        } else {
          mma_bf16_elect(d_tmem, ad + 2u * k, bd + 2u * k, idesc, (first | k) ? 1u : 0u);
        }
      }
    };
    for (int L = t0; L < tot_it; L += tstep) {
      mbar_wait(tempty0 + 8u * acc, aph ^ 1u);
      tc_fence_after();
      // 3xTF32: K step i of the tile accumulates into partial accumulator i % G (G = nsplit), so no
      // fp32 accumulation chain in TMEM is longer than K / (8 G) MMAs (the tensor core's fp32 adds
      // are not round-to-nearest: their error grows with the chain, tools/x3_accuracy.py)
      const int G = X3 ? P.nsplit : 1;
      const uint32_t d_base = tmem_base + (uint32_t)(acc * BN * G);
      if (HALO) {
        for (int ch = 0; ch < g.nchunk; ++ch) {
          mbar_wait(ready0 + 8u * s, ph);
          tc_fence_after();
          const uint64_t dh = dA0 + ((s * op_a) >> 4);
          for (int tap = 0; tap < 9; ++tap) {
            const uint32_t p0 = (uint32_t)((g.dh[tap] + 1) * (g.Wt + 2) + (g.dw[tap] + 1));
            const uint64_t ad = dh + ((p0 * (uint32_t)KB) >> 4);
            uint64_t bd;
            if (STREAMB) {
              if (!TCX_NO_B) mbar_wait(fullB0 + 8u * sb, phb);
              tc_fence_after();
              bd = dB0 + (((uint32_t)sb * bslot) >> 4);
            } else {
              bd = dB0 + (((uint32_t)(tap * g.nchunk + ch) * b_stage) >> 4);
            }
            const int i = ch * 9 + tap;
            mma_k(d_base + (uint32_t)((i % G) * BN), ad, bd, (uint32_t)(i >= G));
            if (STREAMB) {
              if (!TCX_NO_B) mma_commit_elect(emptyB0 + 8u * sb);
              if (++sb == SB) { sb = 0; phb ^= 1u; }
            }
          }
          mma_commit_elect(empty0 + 8u * s);
          if (++s == S) { s = 0; ph ^= 1u; }
        }
      } else {
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(ready0 + 8u * s, ph);
          if (X3) mbar_wait(full0 + 8u * s, ph);  // the B boxes of the stage (same transaction)
          tc_fence_after();
          mma_k(d_base + (uint32_t)((kb % G) * BN), dA0 + ((s * a_stage) >> 4), dB0 + ((s * bslot) >> 4),
                (uint32_t)(kb >= G));
          mma_commit_elect(empty0 + 8u * s);
          if (++s == S) { s = 0; ph ^= 1u; }
        }
      }
      mma_commit_elect(tfull0 + 8u * acc);
      if (++acc == NA) { acc = 0; aph ^= 1u; }
    }
  } else if (warp >= 2 && warp < 10) {
    // ---------------- epilogue warps 2..9: TMEM lane quadrant = warp % 4, one pixel row per
    // thread; the two warps of a quadrant split the tile's columns in halves. Each quadrant
    // publishes its own 32-row slab (pair barrier of 64 threads + one TMA store per column box),
    // so no warp waits for the whole tile or for a store to drain: the slab's leader releases
    // the epilogue buffer of the PREVIOUS tile once that tile's stores have been read.
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int row = quad * 32 + lane;
    const bool qleader = (half == 0 && lane == 0);
    const int cbeg = half * (BN >> 1), cend = cbeg + (BN >> 1);
    const bool slab_live = quad * 32 < g.R * g.Wt;
    // slab mode: 4 storers (one per quadrant); whole-tile mode (Wt neither a multiple nor a divisor
    // of 32, e.g. ragged test shapes): warp 2 stores the tile after an 8-warp barrier
    const bool storer = P.slab_mode ? qleader : (qleader && quad == 2);
    const uint32_t arrivals = P.slab_mode ? 1u : 4u;
    // slab origin inside the tile (pixel rows of the M tile are row-major R x Wt)
    const int sh = (quad * 32) / g.Wt, sw = (quad * 32) % g.Wt;
    int acc = 0, eb = 0, prev_eb = -1;  // accumulator stage, epilogue buffer
    uint32_t aph = 0, eph = 0;
    for (int L = t0; L < tot_it; L += tstep) {
      const TileIdx ti = tile_index(P, live_tile(P, L));
      const int img = ti.img, h0 = ti.h0, w0 = ti.w0, nt = ti.nt;
      const uint32_t ebuf = sE + eb * epi_stage;
      if (HAS_AUX) {
        mbar_wait(auxfull0 + 8u * eb, eph);
      } else {
        mbar_wait(epifree0 + 8u * eb, eph ^ 1u);
      }
      mbar_wait(tfull0 + 8u * acc, aph);
      tc_fence_after();
      if (TCX_NO_EPI) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty0 + 8u * acc);
        if (qleader) mbar_arrive(epifree0 + 8u * eb);  // 4 arrivals
        if (++acc == NA) { acc = 0; aph ^= 1u; }
        if (++eb == NE) { eb = 0; eph ^= 1u; }
        continue;
      }
      if (EPI == EPI_IMG) {
        // image planes straight from TMEM: the warps of the first column half own columns 0..15
        if (half == 0) {
          float v[16];
          tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * BN), v);
          const int oh = h0 + row / g.Wt, ow = w0 + row % g.Wt;
          if (row < g.R * g.Wt && oh < g.OH && ow < g.OW) {
            const long long plane = (long long)g.OH * g.OW;
            const long long o = (long long)img * P.img_c * plane + (long long)oh * g.OW + ow;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              if (c < P.img_c) {
                const float a = P.img_aux ? P.img_alpha * P.img_aux[o + c * plane] : 0.f;
                P.img_out[o + c * plane] = v[c] + a;
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty0 + 8u * acc);
        if (qleader) mbar_arrive(epifree0 + 8u * eb);  // 4 arrivals, nothing stored through smem
        if (++acc == NA) { acc = 0; aph ^= 1u; }
        if (++eb == NE) { eb = 0; eph ^= 1u; }
        continue;
      }
      const int G = X3 ? P.nsplit : 1;
#pragma unroll 1
      for (int c0 = cbeg; c0 < cend; c0 += 16) {
        float v[16];
        const uint32_t tq = tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * BN * G + c0);
        tmem_ld16(tq, v);
        for (int j = 1; j < G; ++j) {  // 3xTF32 partial accumulators, summed in fp32 (RNE)
          float u[16];
          tmem_ld16(tq + (uint32_t)(j * BN), u);
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] += u[e];
        }
        const uint32_t box = ebuf + (uint32_t)(c0 / BOXC) * P.epi_box_bytes;
        constexpr int VPC = 16 / ES;               // values per 16-byte chunk
        const int j0 = ((c0 % BOXC) * ES) >> 4;    // first chunk of these 16 columns in the row
#pragma unroll
        for (int q = 0; q < ES; ++q) {             // 16 columns = ES chunks
          const uint32_t a = epi_chunk_addr<BOXB>(box, row, j0 + q);
          const float* vq = v + q * VPC;
          uint4 w;
          if (X3) {
            float o[4];
            if (HAS_AUX) {
              const uint4 u = ld_shared_v4(a);
              const float f[4] = {__uint_as_float(u.x), __uint_as_float(u.y), __uint_as_float(u.z), __uint_as_float(u.w)};
#pragma unroll
              for (int e = 0; e < 4; ++e) o[e] = (EPI == EPI_RESADD) ? vq[e] + f[e] : vq[e] * dsoftplus_from_act(f[e]);
            } else {
#pragma unroll
              for (int e = 0; e < 4; ++e) o[e] = (EPI == EPI_SOFTPLUS) ? softplus_f(vq[e]) : vq[e];
            }
            w = make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]), __float_as_uint(o[2]), __float_as_uint(o[3]));
          } else {
            float o[8];
            if (HAS_AUX) {
              const uint4 u = ld_shared_v4(a);
              const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h2[e]);
                if (EPI == EPI_RESADD) {
                  o[2 * e] = vq[2 * e] + f.x;
                  o[2 * e + 1] = vq[2 * e + 1] + f.y;
                } else {
                  o[2 * e] = vq[2 * e] * dsoftplus_from_act_fast(f.x);
                  o[2 * e + 1] = vq[2 * e + 1] * dsoftplus_from_act_fast(f.y);
                }
              }
            } else {
#pragma unroll
              for (int e = 0; e < 8; ++e)
                o[e] = (EPI == EPI_SOFTPLUS) ? ((e & 1) ? softplus_poly_log(vq[e]) : softplus_fast(vq[e])) : vq[e];
            }
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
            for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(o[2 * e], o[2 * e + 1]);
          }
          st_shared_v4(a, w);
        }
      }
      // TMEM stage fully read: let the MMA warp reuse it
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(tempty0 + 8u * acc);
      // publish this quadrant's slab: generic-proxy smem writes -> async proxy, pair barrier,
      // then one TMA store per column box of the slab
      fence_async_smem();
      if (P.slab_mode) pair_bar(quad);
      else epi_bar();
      if (storer) {
        if (P.slab_mode) {
          if (slab_live) {
            for (int b = 0; b < nbox; ++b) {
              const int col = nt * BN + b * BOXC;
              tma_store_5d(&tmSlab, ebuf + b * P.epi_box_bytes + (uint32_t)(quad * 32) * BOXB, col % g.CB,
                           w0 + sw, col / g.CB, h0 + sh, img);
            }
          }
        } else {
          for (int b = 0; b < nbox; ++b) {
            const int col = nt * BN + b * BOXC;
            tma_store_5d(&tmOut, ebuf + b * P.epi_box_bytes, col % g.CB, w0, col / g.CB, h0, img);
          }
        }
        bulk_commit();
        // release the previous tile's buffer once its stores have been read
        if (NE == 1) {  // one buffer: released as soon as this tile's stores have read it
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          mbar_arrive_n(epifree0, arrivals);
        } else {
          if (prev_eb >= 0) {
            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            mbar_arrive_n(epifree0 + 8u * prev_eb, arrivals);
          }
          prev_eb = eb;
        }
      }
      if (++acc == NA) { acc = 0; aph ^= 1u; }
      if (++eb == NE) { eb = 0; eph ^= 1u; }
    }
    if (storer) {
      bulk_wait0();
      if (prev_eb >= 0) mbar_arrive_n(epifree0 + 8u * prev_eb, arrivals);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(P.tmem_cols)
                 : "memory");
}

// ------------------------------------------------------------------ fused head (image -> features)
// out[n,h,w,co] = sum_k B[co][k] * patch[n,h,w,k], patch k = c*9 + a*3 + b (c < C <= 3, zero for
// k >= 9C): the C -> NC 3x3 head conv (and the tail adjoint) as ONE kernel. Each thread builds its
// pixel's K = 32 im2col row straight into the swizzled (SW64) shared A tile -- the 134 MB im2col
// tensor of the two-kernel form never touches HBM -- then one elected lane issues two
// M128 x NC x K16 tcgen05.mma into a TMEM accumulator that the same thread reads back with
// tcgen05.ld (thread = pixel = TMEM lane) and stores as 16-byte bf16 chunks (a warp writes 32
// consecutive pixels = one contiguous run). The output staging is double-buffered
// (asynchronous tensor stores); A and the accumulator are single (the loop waits for each MMA),
// which lets 8 CTAs share an SM to hide the per-tile round trip.
template <int NC>
__global__ void __launch_bounds__(128) img2feat_tc_kernel(const float* __restrict__ in,
                                                          const __nv_bfloat16* __restrict__ wB,
                                                          const __grid_constant__ CUtensorMap tmO, int N, int C,
                                                          int H, int W, const FastDiv fdHW, const FastDiv fdW,
                                                          const int* __restrict__ act_list, const int* n_act) {
  // ONE static array carved by hand (A tile | B tile | output staging | barriers | TMEM address):
  // separate 1024-aligned arrays get padded to 28 / 46 KB, and a dynamic staging buffer needs 1 KB
  // of alignment slack -- either costs one resident CTA per SM (8 fit at NC = 32; NC = 64 fits 4 either way).
  // Output staging [2][128 pixels x NC] is in the TMA store's swizzle (SW64 for NC = 32, SW128 for
  // 64): conflict-free 16-byte writes (a linear layout at a 64/128-byte pixel stride put 8 lanes
  // on 2 / 1 bank groups), un-swizzled by the TMA tensor store
  constexpr int SM_A = 128 * 64, SM_B = NC * 64, SM_O = 2 * 128 * NC * 2;
  __shared__ __align__(1024) unsigned char smem_all[SM_A + SM_B + SM_O + 32];
  unsigned char* const sAraw = smem_all;                 // one A tile: the loop waits for each MMA
  unsigned char* const sBraw = smem_all + SM_A;
  unsigned char* const sOdyn = smem_all + SM_A + SM_B;
  uint64_t* const bar = reinterpret_cast<uint64_t*>(smem_all + SM_A + SM_B + SM_O);
  uint32_t& tmem_holder = *reinterpret_cast<uint32_t*>(smem_all + SM_A + SM_B + SM_O + 16);
  const int tid = threadIdx.x;
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  const uint32_t sA = smem_u32(sAraw), sB = smem_u32(sBraw);
  // weights [NC][32] bf16 -> swizzled K-major B tile (64-byte rows, 16-byte chunk j at j ^ ((r >> 1) & 3))
  for (int i = tid; i < NC * 4; i += 128) {
    const int r = i >> 2, j = i & 3;
    const uint4 v = *reinterpret_cast<const uint4*>(wB + r * 32 + j * 8);
    st_shared_v4(sB + (uint32_t)r * 64u + (uint32_t)((j ^ ((r >> 1) & 3)) << 4), v);
  }
  if (tid == 0) {
    mbar_init(smem_u32(&bar[0]), 1);
    mbar_init(smem_u32(&bar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_holder)),
                 "r"((uint32_t)NC)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, tmem_holder, 0);
  // programmatic dependent launch: the prologue above (weights, barriers, TMEM) overlapped the
  // previous kernel; the image and the active flags are read only after it completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const long long HW = (long long)H * W, total = (long long)N * HW;
  const long long tiles = (total + 127) / 128;
  const uint32_t idesc = make_idesc_bf16(NC);
  const uint64_t dB = make_sdesc(sB, 512u, 4u);
  // 32-bit pixel indexing (N*H*W < 2^31 for every supported size) with multiply-shift division
  // the patch of the NEXT tile is loaded into registers before this tile's MMA/epilogue, so the
  // global-load latency overlaps the tensor-core round trip and the staging of the output
  float pv[27];
  auto load_patch = [&](long long tt) {
    const long long px = tt * 128 + tid;
#pragma unroll
    for (int k = 0; k < 27; ++k) pv[k] = 0.f;
    if (px < total) {
      const uint32_t p32 = (uint32_t)px;
      const uint32_t n = fdHW.div(p32), rem = p32 - n * (uint32_t)HW;
      const uint32_t h = fdW.div(rem), w = rem - h * (uint32_t)W;
      if (h >= 1 && h + 1 < (uint32_t)H && w >= 1 && w + 1 < (uint32_t)W) {
        // interior pixel (all but the image border): one base pointer, 27 loads at fixed offsets
        const float* p0 = in + ((long long)n * C) * HW + (long long)(h - 1) * W + (w - 1);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (c < C) {
            const float* pc = p0 + (long long)c * HW;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
              for (int b = 0; b < 3; ++b) pv[c * 9 + a * 3 + b] = __ldg(pc + a * W + b);
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          if (c < C) {
            const float* plane = in + ((long long)n * C + c) * HW;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
              for (int b = 0; b < 3; ++b) {
                const int hh = (int)h + a - 1, ww = (int)w + b - 1;
                if (hh >= 0 && hh < H && ww >= 0 && ww < W) pv[c * 9 + a * 3 + b] = __ldg(plane + hh * W + ww);
              }
          }
        }
      }
    }
  };
  // early-stopping solves: walk only the tiles of the active images (the solver's compacted
  // list; images are whole 128-pixel tiles when H*W % 128 == 0, else every tile is computed)
  const long long tpi = HW / 128;
  const bool use_list = act_list != nullptr && (HW % 128) == 0;
  const long long nlog = use_list ? (long long)(*(volatile const int*)n_act) * tpi : tiles;
  auto raw_tile = [&](long long L) -> long long {
    if (!use_list) return L;
    const long long q = L / tpi;
    return (long long)__ldg(act_list + q) * tpi + (L - q * tpi);
  };
  int it = 0;
  long long t_prev = -1;
  long long Lnext = blockIdx.x;
  if (Lnext < nlog) load_patch(raw_tile(Lnext));
  for (long long L = Lnext; L < nlog; L = Lnext, ++it) {
    Lnext = L + gridDim.x;
    const long long t = raw_tile(L);
    const int buf = it & 1;  // output staging buffer (the only double-buffered resource)
    float v[32];
#pragma unroll
    for (int k = 0; k < 27; ++k) v[k] = pv[k];
#pragma unroll
    for (int k = 27; k < 32; ++k) v[k] = 0.f;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      uint4 wv;
      __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&wv);
#pragma unroll
      for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(v[j * 8 + 2 * e], v[j * 8 + 2 * e + 1]);
      st_shared_v4(sA + (uint32_t)tid * 64u + (uint32_t)((j ^ ((tid >> 1) & 3)) << 4), wv);
    }
    fence_async_smem();  // A tile (and the previous tile's output staging) -> async proxy
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // the next tile's patch loads are issued only now: the proxy fence above (MEMBAR.ALL.CTA)
    // waits for every outstanding load of the thread, so loads issued before it would stall it;
    // from here they overlap the MMA round trip and this tile's epilogue
    if (Lnext < nlog) load_patch(raw_tile(Lnext));
    if (tid == 0) {
      if (t_prev >= 0) {  // the previous tile's staged output: one TMA tensor store (rows past the end clipped)
        tma_store_2d(&tmO, smem_u32(sOdyn + (buf ^ 1) * 128 * NC * 2), 0, (int)(t_prev * 128));
        bulk_commit();
      }
      // the staging buffer this tile writes was bulk-copied one tile ago: wait until it was read
      asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    }
    const uint32_t d_tmem = tmem_base;
    if (warp == 0) {
      const uint64_t dA = make_sdesc(sA, 512u, 4u);
      mma_bf16_elect(d_tmem, dA, dB, idesc, 0u);
      mma_bf16_elect(d_tmem, dA + 2u, dB + 2u, idesc, 1u);
      mma_commit_elect(smem_u32(&bar[0]));
    }
    mbar_wait(smem_u32(&bar[0]), (uint32_t)(it & 1));
    __syncthreads();  // thread 0 has waited for the staging buffer's previous bulk copy
    tc_fence_after();
    const uint32_t so = smem_u32(sOdyn + buf * 128 * NC * 2);
#pragma unroll
    for (int c0 = 0; c0 < NC; c0 += 16) {
      float r[16];
      tmem_ld16(tmem_base + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, r);
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        uint4 wv;
        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&wv);
#pragma unroll
        for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(r[q * 8 + 2 * e], r[q * 8 + 2 * e + 1]);
        st_shared_v4(epi_chunk_addr<NC * 2>(so, tid, c0 / 8 + q), wv);
      }
    }
    tc_fence_before();
    t_prev = t;
  }
  fence_async_smem();
  __syncthreads();
  if (tid == 0) {
    if (t_prev >= 0) {
      tma_store_2d(&tmO, smem_u32(sOdyn + ((it - 1) & 1) * 128 * NC * 2), 0, (int)(t_prev * 128));
      bulk_commit();
    }
    bulk_wait0();
  }
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"((uint32_t)NC)
                 : "memory");
}

// ------------------------------------------------------------------ host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// output [pixels][NC] bf16 as a 2-D tensor, 128-pixel boxes in the staging swizzle (encoded once,
// when the program is built)
struct I2FPlan { CUtensorMap tmO; };
I2FPlan* img2feat_make_plan(__nv_bfloat16* out, int N, int H, int W, int NC, char* err, size_t errlen) {
  EncodeTiledFn enc = get_encode();
  if (!enc) { snprintf(err, errlen, "cuTensorMapEncodeTiled unavailable"); return nullptr; }
  I2FPlan* p = new I2FPlan();
  const long long total = (long long)N * H * W;
  cuuint64_t dims[2] = {(cuuint64_t)NC, (cuuint64_t)total};
  cuuint64_t strides[1] = {(cuuint64_t)NC * 2};
  cuuint32_t box[2] = {(cuuint32_t)NC, 128u};
  cuuint32_t es[2] = {1, 1};
  const CUresult r = enc(&p->tmO, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, out, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, NC == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { snprintf(err, errlen, "img2feat output tensor map encode failed (%d)", (int)r); delete p; return nullptr; }
  return p;
}
void img2feat_free_plan(I2FPlan* p) { delete p; }

// resident img2feat CTAs per SM (0 = not known yet), from the kernel's attributes: shared memory
// (static + the per-block reserve) against the SM's 228 KB, registers (allocated in units of 8 per
// thread), and the 512 TMEM columns. The runtime's occupancy calculator is of no use here: it
// answers 1 for a kernel that allocates TMEM (tools/occ_probe.cu), while ncu's launch__occupancy
// limits agree with this count (8 at NC = 32, 4 at NC = 64). Filled by init_attrs_tc().
static int i2f_occ[2] = {0, 0};
static int img2feat_residency(int NC) {
  cudaFuncAttributes a;
  const cudaError_t e = NC == 64 ? cudaFuncGetAttributes(&a, img2feat_tc_kernel<64>)
                                 : cudaFuncGetAttributes(&a, img2feat_tc_kernel<32>);
  if (e != cudaSuccess) { cudaGetLastError(); return 0; }
  int dev = 0, smem_sm = 0, reserve = 0, regs_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
  cudaDeviceGetAttribute(&reserve, cudaDevAttrReservedSharedMemoryPerBlock, dev);
  cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev);
  if (smem_sm <= 0 || regs_sm <= 0) return 0;
  const int by_smem = smem_sm / ((int)a.sharedSizeBytes + reserve);
  const int by_regs = regs_sm / (((a.numRegs + 7) / 8 * 8) * 128);
  const int by_tmem = 512 / NC;
  const int o = by_smem < by_regs ? by_smem : by_regs;
  return o < 1 ? 0 : (o > by_tmem ? by_tmem : o);
}

void launch_img2feat_tc(const I2FPlan* plan, const float* in, const __nv_bfloat16* wB, const int* act_list,
                        const int* n_act, int N, int C,
                        int H, int W, int NC, int num_sms, cudaStream_t s) {
  // one wave of resident CTAs (each walks tiles at a grid stride): a grid above the residency
  // (8 CTAs per SM at NC = 32, 4 at NC = 64, img2feat_residency) leaves a second, partial wave that
  // starts only when a first-wave CTA retires -- the earlier 8 / 5 per SM ran 7 / 4 + a tail wave
  int per_sm = i2f_occ[NC == 64];
  if (per_sm == 0) per_sm = i2f_occ[NC == 64] = img2feat_residency(NC);
  if (per_sm == 0) per_sm = NC == 64 ? 4 : 8;  // attributes unavailable: ncu's residency for this layout
  const size_t pad = 0;
  const long long total = (long long)N * H * W, tiles = (total + 127) / 128;
  const long long cap = (long long)num_sms * per_sm;
  const unsigned grid = (unsigned)(tiles < cap ? tiles : cap);
  FastDiv fdHW, fdW;
  fdHW.init((uint32_t)(H * W));
  fdW.init((uint32_t)W);
  if (NC == 64)
    launch_k(img2feat_tc_kernel<64>, grid, 128, pad, s, in, wB, plan->tmO, N, C, H, W, fdHW, fdW, act_list, n_act);
  else
    launch_k(img2feat_tc_kernel<32>, grid, 128, pad, s, in, wB, plan->tmO, N, C, H, W, fdHW, fdW, act_list, n_act);
}

struct TcPlan {
  const int* list_ptr;  // the solver's compacted active-image list (tile skipping)
  CUtensorMap tmA, tmB, tmOut, tmAux, tmSlab, tmBlo;
  TcParams P;
  int KB, epi, boxb, grid, halo;
  bool x3;
  size_t smem;
};

// N tile: up to 128 columns (bf16); 32 in 3xTF32 (fp32 staging and the hi / lo operand pairs
// double every shared-memory buffer, and each tile keeps up to 8 partial accumulators in TMEM)
static int tc_bn(const ConvGeom& g, bool x3) {
  const int cap = x3 ? 32 : 128;
  return g.ncols >= cap ? cap : g.ncols;
}

bool tc_supported(const ConvGeom& g, bool x3) {
  if (x3 ? g.KC != 32 : !(g.KC == 32 || g.KC == 64)) return false;
  if (g.R * g.Wt > 128 || g.Wt > 256 || g.R > 256) return false;
  if (x3 && g.epi == EPI_IMG) return false;  // the fp32 mode's head / tail run on the FFMA path
  // EPI_IMG (tail / head adjoint: C <= 3 image columns) runs with N = 16; its epilogue writes
  // fp32 planes from registers and never uses the smem boxes / store maps
  if (g.epi == EPI_IMG ? (g.ncols != 16 && g.ncols != 32) : (g.ncols % 32 != 0)) return false;
  const int BN = tc_bn(g, x3);
  if (g.ncols % BN != 0) return false;
  const int boxc = x3 ? 32 : (BN >= 64 ? 64 : 32);
  if (g.epi != EPI_IMG && (g.CB % boxc != 0 || g.OCp % 8 != 0)) return false;
  if ((g.inC * 2) % 16 != 0) return false;
  if (g.OHo % g.osh != 0) return false;
  return true;
}

// Halo variants: 3x3 taps (|dh|,|dw| <= 1, no parity planes) on tiles whose 8-row core groups
// sit at a uniform stride inside the halo box: 16 x 8 pixels (preferred: 1.4x halo) or one row of
// 128 pixels. Returns 0 (plain), 1 (resident weights) or 2 (streamed weights) and the tile shape.
static int tc_halo_mode(const ConvGeom& g, bool x3, int& R, int& Wt) {
  if (g.ntaps != 9 || g.inP != 1) return 0;
  for (int t = 0; t < 9; ++t)
    if (g.dp[t] != 0 || g.dh[t] < -1 || g.dh[t] > 1 || g.dw[t] < -1 || g.dw[t] > 1) return 0;
  if (g.OW % 8 == 0) { R = 16; Wt = 8; }
  else if (g.R == 1 && g.Wt == 128) { R = 1; Wt = 128; }
  else return 0;
  const int BN = tc_bn(g, x3);
  const size_t wbytes = (size_t)9 * g.nchunk * BN * g.KC * (x3 ? 8 : 2);  // hi (+ lo)
  if (g.ncols == BN && wbytes <= 80 * 1024) return 1;
  return 2;
}

// 5-D view (c, w, p, h, n) of an NHWC tensor of es-byte elements: dims {C, W, P, H, N} (P parity
// planes interleaved in h)
static CUresult encode5(EncodeTiledFn enc, CUtensorMap* m, const void* ptr, int es, int C, int W, int P, int H, int N,
                        int boxc, int boxw, int boxh, CUtensorMapSwizzle sw) {
  cuuint64_t dims[5] = {(cuuint64_t)C, (cuuint64_t)W, (cuuint64_t)P, (cuuint64_t)H, (cuuint64_t)N};
  cuuint64_t strides[4];
  strides[0] = (cuuint64_t)C * es;
  strides[1] = strides[0] * W;
  strides[2] = strides[1] * P;
  strides[3] = strides[2] * H;
  cuuint32_t box[5] = {(cuuint32_t)boxc, (cuuint32_t)boxw, 1u, (cuuint32_t)boxh, 1u};
  cuuint32_t es5[5] = {1, 1, 1, 1, 1};
  return enc(m, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, const_cast<void*>(ptr),
             dims, strides, box, es5, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

static CUresult encode_w(EncodeTiledFn enc, CUtensorMap* m, const void* w, int es, const ConvGeom& g, int BN,
                         CUtensorMapSwizzle sw) {
  const int nkb = g.ntaps * g.nchunk;
  cuuint64_t dims[3] = {(cuuint64_t)g.KC, (cuuint64_t)g.ncols, (cuuint64_t)nkb};
  cuuint64_t strides[2] = {(cuuint64_t)g.KC * es, (cuuint64_t)g.KC * es * g.ncols};
  cuuint32_t box[3] = {(cuuint32_t)g.KC, (cuuint32_t)BN, 1u};
  cuuint32_t e3[3] = {1, 1, 1};
  return enc(m, es == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(w),
             dims, strides, box, e3, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

TcPlan* tc_make_plan(const ConvGeom& g_in, bool x3, const void* in, const void* wB, const void* wBlo, void* out,
                     const void* aux, int num_sms, char* err, size_t errlen) {
  if (!tc_supported(g_in, x3)) { snprintf(err, errlen, "tcgen05 conv: unsupported geometry"); return nullptr; }
  if (x3 && !wBlo) { snprintf(err, errlen, "3xTF32 conv needs the lo weights"); return nullptr; }
  ConvGeom g = g_in;
  EncodeTiledFn enc = get_encode();
  if (!enc) { snprintf(err, errlen, "cuTensorMapEncodeTiled unavailable"); return nullptr; }
  const bool has_aux = g.epi == EPI_RESADD || g.epi == EPI_SIGMUL;
  if (has_aux && !aux) { snprintf(err, errlen, "epilogue needs an aux tensor"); return nullptr; }
  TcPlan* p = new TcPlan();
  memset(p, 0, sizeof(TcPlan));
  const int es = x3 ? 4 : 2;
  const int nbuf = x3 ? 2 : 1;
  p->x3 = x3;
  p->KB = g.KC * es;
  p->epi = g.epi;
  const int BN = tc_bn(g, x3);
  const int boxc = x3 ? 32 : (BN >= 64 ? 64 : 32);
  p->boxb = boxc * es;
  const CUtensorMapSwizzle swA = p->KB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  const CUtensorMapSwizzle swE = p->boxb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B;
  int hR = g.R, hW = g.Wt;
  p->halo = tc_halo_mode(g, x3, hR, hW);
  if (p->halo) {  // halo tiles may re-shape the M tile (16 x 8 pixels)
    g.R = hR;
    g.Wt = hW;
    g.tiles_h = (g.OH + g.R - 1) / g.R;
    g.tiles_w = (g.OW + g.Wt - 1) / g.Wt;
  }
  CUresult r = p->halo ? encode5(enc, &p->tmA, in, es, g.inC, g.inW, g.inP, g.inH, g.N, g.KC, g.Wt + 2, g.R + 2, swA)
                       : encode5(enc, &p->tmA, in, es, g.inC, g.inW, g.inP, g.inH, g.N, g.KC, g.Wt, g.R, swA);
  if (r != CUDA_SUCCESS) { snprintf(err, errlen, "tensor map A encode failed (%d)", (int)r); delete p; return nullptr; }
  r = encode_w(enc, &p->tmB, wB, es, g, BN, swA);
  if (r == CUDA_SUCCESS) r = encode_w(enc, &p->tmBlo, x3 ? wBlo : wB, es, g, BN, swA);
  if (r != CUDA_SUCCESS) { snprintf(err, errlen, "tensor map B encode failed (%d)", (int)r); delete p; return nullptr; }
  const int slab_mode = (g.Wt % 32 == 0 || 32 % g.Wt == 0) ? 1 : 0;
  if (g.epi == EPI_IMG) {  // no smem-staged output: the store / aux / slab maps are never used
    p->tmOut = p->tmA;
    p->tmAux = p->tmA;
    p->tmSlab = p->tmA;
  } else {
    // output / aux: 5-D view (CB, OWo, osh, OHo/osh, N) -- plain NHWC store (osh = 1) or the
    // 2x2 pixel scatter of the transposed / adjoint strided convs (osh = 2, CB = 2 x channels)
    r = encode5(enc, &p->tmOut, out, es, g.CB, g.OWo, g.osh, g.OHo / g.osh, g.N, boxc, g.Wt, g.R, swE);
    if (r != CUDA_SUCCESS) { snprintf(err, errlen, "tensor map out encode failed (%d)", (int)r); delete p; return nullptr; }
    if (has_aux) {
      r = encode5(enc, &p->tmAux, aux, es, g.CB, g.OWo, g.osh, g.OHo / g.osh, g.N, boxc, g.Wt, g.R, swE);
      if (r != CUDA_SUCCESS) { snprintf(err, errlen, "tensor map aux encode failed (%d)", (int)r); delete p; return nullptr; }
    } else {
      p->tmAux = p->tmOut;
    }
    // 32-row epilogue slab (one TMEM lane quadrant): Wt >= 32 -> 32 pixels of one row; Wt < 32 ->
    // 32 / Wt whole rows. Used when Wt is a multiple or a divisor of 32.
    if (slab_mode) {
      const int sw = g.Wt >= 32 ? 32 : g.Wt, sh = g.Wt >= 32 ? 1 : 32 / g.Wt;
      r = encode5(enc, &p->tmSlab, out, es, g.CB, g.OWo, g.osh, g.OHo / g.osh, g.N, boxc, sw, sh, swE);
      if (r != CUDA_SUCCESS) { snprintf(err, errlen, "tensor map slab encode failed (%d)", (int)r); delete p; return nullptr; }
    } else {
      p->tmSlab = p->tmOut;
    }
  }
  TcParams& P = p->P;
  P.g = g;
  P.BN = BN;
  P.n_tiles = g.ncols / BN;
  P.m_tiles = g.N * g.tiles_h * g.tiles_w;
  P.slab_mode = slab_mode;
  P.fd_ntiles.init((uint32_t)P.n_tiles);
  P.fd_perimg.init((uint32_t)(g.tiles_h * g.tiles_w));
  P.fd_tw.init((uint32_t)g.tiles_w);
  P.a_bytes = (uint32_t)p->KB * g.Wt * g.R;
  P.b_bytes = (uint32_t)p->KB * BN;
  P.epi_box_bytes = 128u * (uint32_t)p->boxb;
  P.epi_tx_bytes = (uint32_t)(BN / boxc) * (uint32_t)p->boxb * g.Wt * g.R;
  // Shared-memory / TMEM plan. Preference order: deep accumulator rings for narrow N (more tiles
  // in flight hide the per-tile epilogue latency: 8 stages for the 32-column halo layers measured
  // +0.3..1.6% over 4, 2 stages -22%), then 2 CTAs per SM (bf16), then deeper operand rings.
  const size_t a_stage = 128u * (size_t)p->KB, b_stage = (size_t)BN * p->KB, bslot = b_stage * nbuf,
               e_stage = (size_t)BN * 128u * es;
  const size_t wbytes = p->halo == 1 ? (size_t)9 * g.nchunk * bslot : 0;
  if (p->halo) {
    P.a_bytes = (uint32_t)p->KB * (g.Wt + 2) * (g.R + 2);
    P.halo_stage = (P.a_bytes + 1023u) & ~1023u;
  }
  // MODE 2: a weight ring of SB slots (one (chunk, tap) box pair each) next to the halo ring
  const int SBq = x3 ? 3 : 6;
  const bool streamb = p->halo == 2;
  size_t bring = streamb ? (size_t)SBq * bslot : 0;
  P.stagesB = streamb ? SBq : 0;
  const size_t op_stage = p->halo ? (size_t)P.halo_stage * nbuf : a_stage * nbuf + bslot;
  // short-K layers (the 2x2 up / down scatters: 1-2 K-blocks per tile) are bound by the per-tile
  // epilogue round trip (aux load, store), so they take 4 accumulator/epilogue stages and only the
  // operand stages one tile needs
  const int nkb_tile = p->halo ? g.nchunk : g.ntaps * g.nchunk;
  const bool short_k = !p->halo && nkb_tile <= 2;
  const int min_stages = p->halo ? 2 : (short_k ? 2 : 3), max_stages = p->halo ? 4 : (short_k ? 4 : 8);
  int stages = 0, ctas = 1, nacc = 0;
  uint32_t tcols = 0;
  // 3xTF32: up to 8 partial accumulators per tile (one per K step of the tile, cyclically)
  const int ksteps = p->halo ? 9 * g.nchunk : g.ntaps * g.nchunk;
  P.nsplit = x3 ? (ksteps < 8 ? ksteps : 8) : 1;
  const uint32_t acc_w = (uint32_t)BN * P.nsplit;  // TMEM columns per stage
  const int na0 = (8 * acc_w <= 256 && p->halo) ? 8 : ((BN <= 64 || short_k) && 4 * acc_w <= 512 ? 4 : 2);
  const size_t nbar = 64 * 8 + 64;  // barriers and the TMEM holder
  for (int na = na0; na >= 2 && !stages; na -= 2) {
    uint32_t tc = 32;
    while (tc < (uint32_t)na * acc_w) tc <<= 1;
    const size_t fixed = 1024 + (size_t)na * e_stage + wbytes + bring + nbar;
    for (int c = x3 ? 1 : 2; c >= 1 && !stages; --c) {
      const size_t avail = c == 2 ? (227 * 1024) / 2 - 1024 : 220 * 1024;
      if (tc * c > 512 || avail <= fixed) continue;
      int st = (int)((avail - fixed) / op_stage);
      if (st > max_stages) st = max_stages;
      if (st >= min_stages || (c == 1 && na == 2 && st >= 2)) { stages = st; ctas = c; nacc = na; tcols = tc; }
    }
  }
  if (!stages) { snprintf(err, errlen, "tcgen05 conv: shared memory plan failed"); delete p; return nullptr; }
  // streamed-weight layers (bf16): one epilogue buffer (released as soon as its TMA stores have read
  // it) and the freed shared memory added to the weight ring -- the ring's lookahead in time is what
  // bounds these layers (profiles/r2c_conv_bisect.txt: the weight stream costs ~5 us per launch)
  int nepi = nacc;
  if (streamb && !x3 && ctas == 1 && nacc >= 2) {
    nepi = 1;
    const int extra = (int)(((size_t)(nacc - 1) * e_stage) / bslot);
    P.stagesB = SBq + extra > 12 ? 12 : SBq + extra;
    bring = (size_t)P.stagesB * bslot;
  }
  P.stages = stages;
  P.nacc = nacc;
  P.nepi = nepi;
  P.tmem_cols = tcols;
  p->smem = 1024 + (size_t)nepi * e_stage + wbytes + bring + nbar + (size_t)stages * op_stage;
  const int total = P.m_tiles * P.n_tiles;
  const int maxg = num_sms * ctas;
  p->grid = total < maxg ? total : maxg;
  return p;
}

// Every conv launch carries the programmatic-stream-serialization attribute (PDL): it may start
// while its predecessor drains; the kernel waits (griddepcontrol.wait) before reading activations.
template <int KB, int EPI, int BOXB, bool X3>
static void launch_one(const TcPlan* p, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p->grid);
  cfg.blockDim = dim3(X3 ? TC_THREADS_X3 : TC_THREADS);
  cfg.dynamicSmemBytes = p->smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  switch (p->halo) {
    case 1: cudaLaunchKernelEx(&cfg, conv_tc_kernel<KB, EPI, BOXB, 1, X3>, p->tmA, p->tmB, p->tmOut, p->tmAux, p->tmSlab, p->tmBlo, p->P); break;
    case 2: cudaLaunchKernelEx(&cfg, conv_tc_kernel<KB, EPI, BOXB, 2, X3>, p->tmA, p->tmB, p->tmOut, p->tmAux, p->tmSlab, p->tmBlo, p->P); break;
    default: cudaLaunchKernelEx(&cfg, conv_tc_kernel<KB, EPI, BOXB, 0, X3>, p->tmA, p->tmB, p->tmOut, p->tmAux, p->tmSlab, p->tmBlo, p->P); break;
  }
}

template <int KB, int BOXB, bool X3>
static void launch_epi(const TcPlan* p, cudaStream_t s) {
  switch (p->epi) {
    case EPI_SOFTPLUS: launch_one<KB, EPI_SOFTPLUS, BOXB, X3>(p, s); break;
    case EPI_RESADD: launch_one<KB, EPI_RESADD, BOXB, X3>(p, s); break;
    case EPI_SIGMUL: launch_one<KB, EPI_SIGMUL, BOXB, X3>(p, s); break;
    case EPI_IMG: if constexpr (!X3) launch_one<KB, EPI_IMG, BOXB, X3>(p, s); break;
    default: launch_one<KB, EPI_STORE, BOXB, X3>(p, s); break;
  }
}

void tc_plan_set_active(TcPlan* p, const int* act_list, const int* n_act) {
  p->list_ptr = act_list;
  p->P.n_act = n_act;
  p->P.act_list = nullptr;
  p->P.tpi = p->P.g.tiles_h * p->P.g.tiles_w * p->P.n_tiles;
  p->P.fd_tpi.init((uint32_t)p->P.tpi);
}

// The live list is switched on only for solves that can freeze images (tol > 0, per-image rule,
// unless the caller asks for every tile); the CUDA graph of each parameter set captures the choice.
void tc_plan_enable_skip(TcPlan* p, bool on) { p->P.act_list = on ? p->list_ptr : nullptr; }

void tc_plan_set_image(TcPlan* p, float* out, const float* aux, float alpha, int C) {
  p->P.img_out = out;
  p->P.img_aux = aux;
  p->P.img_alpha = alpha;
  p->P.img_c = C;
}

void tc_launch(const TcPlan* p, cudaStream_t s) {
  if (p->x3) {
    launch_epi<128, 128, true>(p, s);
  } else if (p->KB == 128) {
    if (p->boxb == 128) launch_epi<128, 128, false>(p, s); else launch_epi<128, 64, false>(p, s);
  } else {
    if (p->boxb == 128) launch_epi<64, 128, false>(p, s); else launch_epi<64, 64, false>(p, s);
  }
}

int tc_plan_is_halo(const TcPlan* p) { return p->halo; }

void tc_free_plan(TcPlan* p) { delete p; }

template <int KB, int BOXB, int HALO, bool X3>
static void attrs_epi() {
  set_max_dyn_smem(conv_tc_kernel<KB, EPI_STORE, BOXB, HALO, X3>);
  set_max_dyn_smem(conv_tc_kernel<KB, EPI_SOFTPLUS, BOXB, HALO, X3>);
  set_max_dyn_smem(conv_tc_kernel<KB, EPI_RESADD, BOXB, HALO, X3>);
  set_max_dyn_smem(conv_tc_kernel<KB, EPI_SIGMUL, BOXB, HALO, X3>);
  if constexpr (!X3) set_max_dyn_smem(conv_tc_kernel<KB, EPI_IMG, BOXB, HALO, X3>);
}

template <int HALO>
static void attrs_mode() {
  attrs_epi<128, 128, HALO, false>();
  attrs_epi<128, 64, HALO, false>();
  attrs_epi<64, 128, HALO, false>();
  attrs_epi<64, 64, HALO, false>();
  attrs_epi<128, 128, HALO, true>();
}

void init_attrs_tc() {
  i2f_occ[0] = img2feat_residency(32);
  i2f_occ[1] = img2feat_residency(64);
  attrs_mode<0>();
  attrs_mode<1>();
  attrs_mode<2>();
}

}  // namespace ideq
