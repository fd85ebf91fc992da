// Residual-block-fused level-0 convolutions (bf16, tcgen05, row streaming).
//
// A residual block of the U-Net (reading Q10) is two 3x3 convolutions at the same width:
//   forward (Eq. 2's network):  a = sp(A t)  (saved for the VJP),  t' = t + B a
//   input VJP (its transpose):           q = (B^T g) . sp'(a),              g' = g + A^T q
// Run as two launches, the intermediate (a or q) makes a round trip through HBM and the block
// input is read twice (conv input, then residual): at level 0 of C3 that is 671 MB per block for
// 403 MB of compulsory traffic. This kernel computes the whole block for full image rows:
//
//   * a CTA owns a run of consecutive output rows of one image and streams down it. Input rows
//     (the block input x = t or g) arrive by TMA into a 4-slot ring of full-width rows with a zero
//     pixel on either side (the convolutions' zero padding at the image's left / right border);
//   * stage 1 computes the intermediate row u (128-pixel M tiles, the 9 taps as row- and pixel-
//     shifted UMMA descriptors into the ring), its epilogue (softplus, or x sp'(a) with the saved
//     activation from a second TMA ring) writes the row in the UMMA operand layout into a 4-slot
//     ring of intermediate rows (forward: and TMA-stores it as the saved activation); rows outside
//     the image are zeros (the second convolution's zero padding);
//   * stage 2 computes the output row from three intermediate rows; its epilogue adds the
//     residual, read from the input ring, writes the result in place over that input row and
//     TMA-stores it.
// HBM traffic per block: read x (+ a in the VJP), write u (forward) and the output: 403 MB at C3.
// Each run recomputes two intermediate rows (h0 - 1 and the row below the last) -- 2 of ~55 rows.
//
// Warp roles (352 threads, one CTA per SM): warp 0 TMA producer, warp 1 TMEM allocator + MMA
// issuer, warps 2..9 epilogue (TMEM lane quadrant = warp % 4, column half = (warp - 2) / 4).
#include <cuda.h>
#include <stdio.h>
#include <string.h>
#include "common.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace ideq {

constexpr int RBF_THREADS = 352;
constexpr int RBF_XS = 4, RBF_US = 4, RBF_AS = 2;  // ring depths (input rows, intermediate rows, saved act.)
constexpr int RBF_C = 32;                          // channels (64-byte pixels, SW64)
constexpr uint32_t RBF_PIX = RBF_C * 2;

struct RbfParams {
  int N, H, W, MT;            // images, rows, width (= 128 MT)
  int dh1[9], dw1[9], dh2[9], dw2[9];
  uint32_t slot;              // bytes of one ring slot (1 KB pad, zero pixel, W pixels, zero pixel, pad)
  const __nv_bfloat16* w1;    // [9][32][32] GEMM operand of conv 1 / conv 2 (gemm_weights layout)
  const __nv_bfloat16* w2;
  const int* act_list;        // live-image list (null: every image)
  const int* n_act;
  uint32_t tmem_cols;
  int dbg;  // bisection: bit0 no TMA loads, bit1 no MMAs, bit2 no epilogue smem / TMA stores
};

// payload (pixel 0) of a ring slot: 1024-byte aligned; pixel -1 and pixel W are zero forever
__device__ __forceinline__ uint32_t rbf_payload(uint32_t ring, int slot, uint32_t slot_bytes) {
  return ring + (uint32_t)slot * slot_bytes + 1024u;
}
// 16-byte chunk j (8 channels) of pixel p in a payload (the SW64 pattern TMA / UMMA use)
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
__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }

// The CTA's runs: rows [r0, r1) of the (live) row sequence q = image_index * H + h, cut at image
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

__device__ int* g_rbf_prog;  // debug: progress markers in host-mapped memory (null: off)
__device__ __forceinline__ void rbf_mark(int slot, int v) {
  if (g_rbf_prog && blockIdx.x == 0) { ((volatile int*)g_rbf_prog)[slot] = v; __threadfence_system(); }
}

template <bool VJP>
__global__ void __launch_bounds__(RBF_THREADS, 1)
    rbf_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmOut,
               const __grid_constant__ CUtensorMap tmU, const __grid_constant__ RbfParams P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
  unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
  const int W = P.W, MT = P.MT;
  const uint32_t SLOT = P.slot;
  // [weights conv1 9 x 2 KB][weights conv2][x ring][u ring][a ring (VJP)][barriers]
  const uint32_t sW1 = base, sW2 = base + 9u * 2048u;
  const uint32_t sX = base + 18u * 2048u;
  const uint32_t sU = sX + RBF_XS * SLOT;
  const uint32_t sA = sU + RBF_US * SLOT;
  const uint32_t sBar = sA + (VJP ? RBF_AS * SLOT : 0u);
  // barriers: xfull[XS] xempty[XS] ufull[US] uempty[US] afull[AS] aempty[AS] t1full[2] t1empty[2] t2full[2] t2empty[2]
  const uint32_t xfull0 = sBar, xempty0 = xfull0 + 8u * RBF_XS, ufull0 = xempty0 + 8u * RBF_XS,
                 uempty0 = ufull0 + 8u * RBF_US, afull0 = uempty0 + 8u * RBF_US, aempty0 = afull0 + 8u * RBF_AS,
                 t1full0 = aempty0 + 8u * RBF_AS, t1empty0 = t1full0 + 16u, t2full0 = t1empty0 + 16u,
                 t2empty0 = t2full0 + 16u;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(gbase + (t2empty0 + 16u - base));
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  // ---- prologue: weights into the UMMA B layout (rows of 64 bytes, SW64), zero rings, barriers
  for (int i = threadIdx.x; i < ((P.dbg & 16) ? 0 : 2 * 9 * 32 * 4); i += blockDim.x) {
    const int which = i / (9 * 32 * 4), r = (i / 4) % (9 * 32), j = i & 3;  // r = tap * 32 + n
    const __nv_bfloat16* src = (which ? P.w2 : P.w1) + (size_t)r * 32 + j * 8;
    const uint32_t dst = (which ? sW2 : sW1) + (uint32_t)r * 64u + (uint32_t)((j ^ ((r >> 1) & 3)) << 4);
    st_shared_v4(dst, *reinterpret_cast<const uint4*>(src));
  }
  {
    const uint32_t ring_bytes = (RBF_XS + RBF_US + (VJP ? RBF_AS : 0)) * SLOT;
    for (uint32_t o = threadIdx.x * 16u; o < ((P.dbg & 32) ? 0u : ring_bytes); o += blockDim.x * 16u)
      st_shared_v4(sX + o, make_uint4(0u, 0u, 0u, 0u));
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < RBF_XS; ++s) { mbar_init(xfull0 + 8u * s, 1); mbar_init(xempty0 + 8u * s, 2); }
    // uempty: the MMA warp's commit after the row's last use (+ forward: the epilogue once the
    // row's TMA store has read the slot)
    for (int s = 0; s < RBF_US; ++s) { mbar_init(ufull0 + 8u * s, 1); mbar_init(uempty0 + 8u * s, VJP ? 1 : 2); }
    for (int s = 0; s < RBF_AS; ++s) { mbar_init(afull0 + 8u * s, 1); mbar_init(aempty0 + 8u * s, 8); }  // 8 epilogue warps
    for (int s = 0; s < 2; ++s) {
      mbar_init(t1full0 + 8u * s, 1); mbar_init(t1empty0 + 8u * s, 8);
      mbar_init(t2full0 + 8u * s, 1); mbar_init(t2empty0 + 8u * s, 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    prefetch_tmap(&tmX);
    prefetch_tmap(&tmOut);
    prefetch_tmap(&tmU);
  }
  if (warp == 1 && !(P.dbg & 256)) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_holder)),
                 "r"(P.tmem_cols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  fence_async_smem();  // weights and zeroed rings -> async proxy (UMMA / TMA)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_holder, 0);
  if (threadIdx.x == 0) rbf_mark(0, 1);
  if (P.dbg & 128) return;

  // this CTA's rows of the live row sequence
  int nimg = P.N;
  if (P.act_list) nimg = ld_volatile_s32(P.n_act);
  const long long Q = (long long)nimg * P.H;
  const int q0 = (int)(Q * blockIdx.x / gridDim.x), q1 = (int)(Q * (blockIdx.x + 1) / gridDim.x);
  const uint32_t row_bytes = (uint32_t)W * RBF_PIX;
  if (P.dbg & 8192) return;

  if (warp == 0 && !(P.dbg & 1024)) {
    // ---------------- producer: x rows h0-2 .. h1+1 of each run (+ VJP: saved-activation rows
    // h0-1 .. h1), in the order x0 x1 x2 | a0 x3 | a1 x4 | ... so no ring waits on a later load
    uint32_t xc = 0, ac = 0;
    int q = q0;
    RbfRun run;
    auto load_x = [&](int n, int h) {
      const int s = (int)(xc % RBF_XS);
      mbar_wait(xempty0 + 8u * s, ((xc / RBF_XS) & 1u) ^ 1u);
      if (elect_one()) {
        if (P.dbg & 1) mbar_arrive(xfull0 + 8u * s);
        else {
        mbar_expect_tx(xfull0 + 8u * s, row_bytes);
        tma_load_4d(rbf_payload(sX, s, SLOT), &tmX, xfull0 + 8u * s, 0, 0, h, n);  // rows outside: zero fill
        }
      }
      __syncwarp();
      ++xc;
      if (lane == 0) rbf_mark(1, (int)xc);
    };
    auto load_a = [&](int n, int h) {
      const int s = (int)(ac % RBF_AS);
      mbar_wait(aempty0 + 8u * s, ((ac / RBF_AS) & 1u) ^ 1u);
      if (elect_one()) {
        mbar_expect_tx(afull0 + 8u * s, row_bytes);
        tma_load_4d(rbf_payload(sA, s, SLOT), &tmU, afull0 + 8u * s, 0, 0, h, n);
      }
      __syncwarp();
      ++ac;
    };
    while (rbf_next_run(P, q, q1, run)) {
      const int nu = run.h1 - run.h0 + 2;  // intermediate rows h0-1 .. h1
      load_x(run.n, run.h0 - 2);
      load_x(run.n, run.h0 - 1);
      load_x(run.n, run.h0);
      for (int iu = 0; iu < nu; ++iu) {
        if (VJP) load_a(run.n, run.h0 - 1 + iu);
        if (iu + 3 <= nu + 1) load_x(run.n, run.h0 - 2 + iu + 3);
      }
    }
  } else if (warp == 1 && !(P.dbg & 2048)) {
    // ---------------- MMA issuer: S1(h0-1), S1(h0), then S1(r+1), S2(r) for r = h0 .. h1-1
    const uint32_t idesc = make_idesc_bf16(RBF_C);
    const uint64_t dW1 = make_sdesc(sW1, 512u, 4u), dW2 = make_sdesc(sW2, 512u, 4u);
    auto commit = [&](uint32_t bar) {
      if (P.dbg & 512) { if (lane == 0) mbar_arrive(bar); __syncwarp(); }
      else mma_commit_elect(bar);
    };
    uint32_t xc = 0, uc = 0, c1 = 0, c2 = 0;  // running ring / accumulator counters
    int q = q0;
    RbfRun run;
    // A operand of tap (dh, dw), M tile mt: payload of the ring row for dh, shifted by dw pixels
    auto mma_row = [&](uint32_t d, uint32_t ring, uint32_t rc_center, int nring, const int* dh, const int* dw,
                       uint64_t dWb) {
      for (int mt = 0; mt < MT; ++mt) {
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const int s = (int)((rc_center + (uint32_t)(nring + dh[tap])) % (uint32_t)nring);
          const uint32_t a_addr = rbf_payload(ring, s, SLOT) + (uint32_t)((128 * mt + dw[tap]) * (int)RBF_PIX);
          const uint64_t ad = make_sdesc(a_addr, 512u, 4u);
          const uint64_t bd = dWb + (((uint32_t)tap * 2048u) >> 4);
#pragma unroll
          for (int k = 0; k < 2; ++k)
            mma_bf16_elect(d + (uint32_t)(mt * RBF_C), ad + 2u * k, bd + 2u * k, idesc, (tap | k) ? 1u : 0u);
        }
      }
    };
    while (rbf_next_run(P, q, q1, run)) {
      const int nu = run.h1 - run.h0 + 2, no = run.h1 - run.h0;
      const uint32_t xb = xc, ub = uc;  // ring counters of the run's first x / u row
      // S1 of intermediate row iu (image row h0-1+iu) reads x run rows iu .. iu+2
      auto s1 = [&](int iu) {
        mbar_wait(xfull0 + 8u * ((xb + iu + 2) % RBF_XS), ((xb + iu + 2) / RBF_XS) & 1u);
        if (iu == 0) {
          mbar_wait(xfull0 + 8u * (xb % RBF_XS), (xb / RBF_XS) & 1u);
          mbar_wait(xfull0 + 8u * ((xb + 1) % RBF_XS), ((xb + 1) / RBF_XS) & 1u);
        }
        const int acc = (int)(c1 & 1u);
        mbar_wait(t1empty0 + 8u * acc, ((c1 >> 1) & 1u) ^ 1u);
        tc_fence_after();
        const int h = run.h0 - 1 + iu;
        if (h >= 0 && h < P.H && !(P.dbg & 2))
          mma_row(tmem_base + (uint32_t)(acc * MT * RBF_C), sX, xb + iu + 1, RBF_XS, P.dh1, P.dw1, dW1);
        commit(t1full0 + 8u * acc);
        ++c1;
        if (lane == 0) rbf_mark(2, (int)c1);
        // x run row k (k = 0 .. nu + 1) is last read by S1(min(k, nu - 1)); rows that are not output
        // rows of the run (k = 0, 1, nu, nu + 1) get both of their arrivals from here
        auto rel_x = [&](int k) {
          const uint32_t bar = xempty0 + 8u * ((xb + k) % RBF_XS);
          commit(bar);
          if (k < 2 || k >= no + 2) commit(bar);
        };
        if (iu < nu - 1) rel_x(iu);
        else { rel_x(nu - 1); rel_x(nu); rel_x(nu + 1); }
      };
      // S2 of output row io (image row h0+io) reads intermediate run rows io .. io+2
      auto s2 = [&](int io) {
        mbar_wait(ufull0 + 8u * ((ub + io + 2) % RBF_US), ((ub + io + 2) / RBF_US) & 1u);
        if (io == 0) {
          mbar_wait(ufull0 + 8u * (ub % RBF_US), (ub / RBF_US) & 1u);
          mbar_wait(ufull0 + 8u * ((ub + 1) % RBF_US), ((ub + 1) / RBF_US) & 1u);
        }
        const int acc = (int)(c2 & 1u);
        mbar_wait(t2empty0 + 8u * acc, ((c2 >> 1) & 1u) ^ 1u);
        tc_fence_after();
        if (!(P.dbg & 2)) mma_row(tmem_base + (uint32_t)((2 + acc) * MT * RBF_C), sU, ub + io + 1, RBF_US, P.dh2, P.dw2, dW2);
        commit(t2full0 + 8u * acc);
        ++c2;
        if (lane == 0) rbf_mark(3, (int)c2);
        // intermediate run row k is last read by S2(min(k, no - 1))
        if (io < no - 1) commit(uempty0 + 8u * ((ub + io) % RBF_US));
        else
          for (int k = no - 1; k < nu; ++k) commit(uempty0 + 8u * ((ub + k) % RBF_US));
      };
      s1(0);
      s1(1);
      for (int io = 0; io < no; ++io) {
        s1(io + 2);
        s2(io);
      }
      xc += (uint32_t)(nu + 2);
      uc += (uint32_t)nu;
    }
  } else if (warp >= 2 && warp < 10 && !(P.dbg & 4096)) {
    // ---------------- epilogue (same stage order as the MMA warp)
    const int quad = warp & 3, half = (warp - 2) >> 2;
    const bool leader = warp == 2 && lane == 0;
    const int c0 = half * 16;  // this warp's 16 channels
    uint32_t xc = 0, uc = 0, ac = 0, c1 = 0, c2 = 0;
    uint32_t pend_bar = 0;     // leader: slot barrier to release once the previous store has been read
    int q = q0;
    RbfRun run;
    auto store_done = [&](uint32_t bar) {  // leader, after committing a store group
      if (pend_bar) { bulk_wait_read1(); mbar_arrive(pend_bar); }
      pend_bar = bar;
    };
    while (rbf_next_run(P, q, q1, run)) {
      const int nu = run.h1 - run.h0 + 2, no = run.h1 - run.h0;
      const uint32_t xb = xc, ub = uc;
      // E1: intermediate row iu -> u ring
      auto e1 = [&](int iu) {
        const int h = run.h0 - 1 + iu;
        const bool inside = h >= 0 && h < P.H;
        const uint32_t us = (ub + iu) % RBF_US;
        mbar_wait(uempty0 + 8u * us, (((ub + iu) / RBF_US) & 1u) ^ 1u);
        uint32_t apl = 0;
        if (VJP) {
          apl = rbf_payload(sA, (int)(ac % RBF_AS), SLOT);
          mbar_wait(afull0 + 8u * (ac % RBF_AS), (ac / RBF_AS) & 1u);
        }
        const int acc = (int)(c1 & 1u);
        mbar_wait(t1full0 + 8u * acc, (c1 >> 1) & 1u);
        tc_fence_after();
        const uint32_t upl = rbf_payload(sU, (int)us, SLOT);
        for (int mt = 0; mt < ((P.dbg & 8) ? 0 : MT); ++mt) {
          float v[16];
          tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)(acc * MT * RBF_C + mt * RBF_C + c0), v);
          const int p = 128 * mt + quad * 32 + lane;
#pragma unroll
          for (int qq = 0; qq < 2; ++qq) {
            const int j = (c0 >> 3) + qq;
            float o[8];
            if (!inside) {
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] = 0.f;
            } else if (VJP) {  // q = (B^T g) . sp'(a)
              const uint4 u = ld_shared_v4(rbf_chunk(apl, p, j));
              const __nv_bfloat162* h2 = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h2[e]);
                o[2 * e] = v[qq * 8 + 2 * e] * dsoftplus_from_act_fast(f.x);
                o[2 * e + 1] = v[qq * 8 + 2 * e + 1] * dsoftplus_from_act_fast(f.y);
              }
            } else {  // a = sp(A t)
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] = (e & 1) ? softplus_poly_log(v[qq * 8 + e]) : softplus_fast(v[qq * 8 + e]);
            }
            uint4 w;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
            for (int e = 0; e < 4; ++e) h2[e] = __floats2bfloat162_rn(o[2 * e], o[2 * e + 1]);
            st_shared_v4(rbf_chunk(upl, p, j), w);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(t1empty0 + 8u * acc);
          if (VJP) mbar_arrive(aempty0 + 8u * (ac % RBF_AS));  // this warp has read its part of the a row
        }
        ++c1;
        if (VJP) ++ac;
        if (leader) rbf_mark(4, (int)c1);
        fence_async_smem();
        epi_bar();
        if (leader) {
          if (!VJP && inside && !(P.dbg & 4)) {  // the saved activation a (the VJP's sp' input)
            tma_store_4d(&tmU, upl, 0, 0, h, run.n);
            bulk_commit();
            mbar_arrive(ufull0 + 8u * us);
            store_done(uempty0 + 8u * us);
          } else {
            mbar_arrive(ufull0 + 8u * us);
            if (!VJP) mbar_arrive(uempty0 + 8u * us);  // nothing stored: the slot is free for the ring
          }
        }
      };
      // E2: output row io = x run row io + 2 (residual), result written over it and stored
      auto e2 = [&](int io) {
        const uint32_t xs = (xb + io + 2) % RBF_XS;
        mbar_wait(xfull0 + 8u * xs, ((xb + io + 2) / RBF_XS) & 1u);
        const int acc = (int)(c2 & 1u);
        mbar_wait(t2full0 + 8u * acc, (c2 >> 1) & 1u);
        tc_fence_after();
        const uint32_t xpl = rbf_payload(sX, (int)xs, SLOT);
        for (int mt = 0; mt < ((P.dbg & 8) ? 0 : MT); ++mt) {
          float v[16];
          tmem_ld16(tmem_base + ((uint32_t)(quad * 32) << 16) + (uint32_t)((2 + acc) * MT * RBF_C + mt * RBF_C + c0), v);
          const int p = 128 * mt + quad * 32 + lane;
#pragma unroll
          for (int qq = 0; qq < 2; ++qq) {
            const int j = (c0 >> 3) + qq;
            const uint32_t addr = rbf_chunk(xpl, p, j);
            const uint4 u = ld_shared_v4(addr);
            const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&u);
            uint4 w;
            __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&w);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 f = __bfloat1622float2(r2[e]);
              h2[e] = __floats2bfloat162_rn(v[qq * 8 + 2 * e] + f.x, v[qq * 8 + 2 * e + 1] + f.y);
            }
            st_shared_v4(addr, w);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(t2empty0 + 8u * acc);
        ++c2;
        if (leader) rbf_mark(5, (int)c2);
        fence_async_smem();
        epi_bar();
        if (leader) {
          if (P.dbg & 4) mbar_arrive(xempty0 + 8u * xs);
          else {
          tma_store_4d(&tmOut, xpl, 0, 0, run.h0 + io, run.n);
          bulk_commit();
          store_done(xempty0 + 8u * xs);
          }
        }
      };
      e1(0);
      e1(1);
      for (int io = 0; io < no; ++io) {
        e1(io + 2);
        e2(io);
      }
      xc += (uint32_t)(nu + 2);
      uc += (uint32_t)nu;
      // the last output row's slot would otherwise wait for the next run's first store, which
      // needs that slot refilled: release it now
      if (leader && pend_bar) {
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        mbar_arrive(pend_bar);
        pend_bar = 0;
      }
    }
    if (leader) {
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      if (pend_bar) mbar_arrive(pend_bar);
      bulk_wait0();
    }
  }
  if (P.dbg & 16384) return;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1 && !(P.dbg & 256))
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(P.tmem_cols)
                 : "memory");
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
  CUtensorMap tmX, tmOut, tmU;
  RbfParams P;
  const int* list_ptr;
  bool vjp;
  int grid;
  size_t smem;
};

bool rbf_supported(int W, int C) { return C == RBF_C && (W == 128 || W == 256); }

size_t rbf_smem_bytes(int W, bool vjp) {
  const size_t slot = ((size_t)1024 + (size_t)(W + 1) * RBF_PIX + 1023) & ~(size_t)1023;
  return 1024 + 18 * 2048 + (RBF_XS + RBF_US + (vjp ? RBF_AS : 0)) * slot + 256;
}

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
  P.N = N; P.H = H; P.W = W; P.MT = W / 128;
  for (int t = 0; t < 9; ++t) { P.dh1[t] = dh1[t]; P.dw1[t] = dw1[t]; P.dh2[t] = dh2[t]; P.dw2[t] = dw2[t]; }
  P.slot = (uint32_t)(((size_t)1024 + (size_t)(W + 1) * RBF_PIX + 1023) & ~(size_t)1023);
  P.w1 = w1; P.w2 = w2;
  P.tmem_cols = 4 * P.MT * RBF_C <= 128 ? 128 : 256;
  CUresult r = rbf_map(enc, &p->tmX, x, N, H, W);
  if (r == CUDA_SUCCESS) r = rbf_map(enc, &p->tmOut, out, N, H, W);
  if (r == CUDA_SUCCESS) r = rbf_map(enc, &p->tmU, act, N, H, W);
  if (r != CUDA_SUCCESS) { snprintf(err, errlen, "fused residual block: tensor map encode failed (%d)", (int)r); delete p; return nullptr; }
  p->smem = rbf_smem_bytes(W, vjp);
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
void rbf_set_debug(RbfPlan* p, int dbg) {
  p->P.dbg = dbg;
  static int* prog = nullptr;
  if (dbg && !prog) {
    int* hp = nullptr;
    if (cudaHostAlloc(&hp, 64 * sizeof(int), cudaHostAllocMapped) == cudaSuccess) {
      memset(hp, 0, 64 * sizeof(int));
      int* dp = nullptr;
      cudaHostGetDevicePointer(&dp, hp, 0);
      cudaMemcpyToSymbol(g_rbf_prog, &dp, sizeof(dp));
      prog = hp;
    }
  }
  if (prog) {
    fprintf(stderr, "rbf progress (previous launch): ");
    for (int i = 0; i < 6; ++i) fprintf(stderr, "%d ", prog[i]);
    fprintf(stderr, "\n");
  }
}


void rbf_launch(const RbfPlan* p, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)p->grid);
  cfg.blockDim = dim3(RBF_THREADS);
  cfg.dynamicSmemBytes = p->smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (p->P.dbg & 64) return;
  if (p->vjp) cudaLaunchKernelEx(&cfg, rbf_kernel<true>, p->tmX, p->tmOut, p->tmU, p->P);
  else cudaLaunchKernelEx(&cfg, rbf_kernel<false>, p->tmX, p->tmOut, p->tmU, p->P);
}

void init_attrs_rbf() {
  set_max_dyn_smem(rbf_kernel<false>);
  set_max_dyn_smem(rbf_kernel<true>);
}

}  // namespace ideq
