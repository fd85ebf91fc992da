/*
 * ideq_debug.h -- test hooks of libideq.so (not needed by solver users).
 *
 * ideq_debug_conv runs ONE implicit-GEMM convolution layer of the network program
 * exactly as the solver does (same weight re-arrangement, geometry and kernel),
 * so tests can pin each layer kind and epilogue against the oracle's layer.
 *
 *   kind 0: conv3x3            out[co,m,n]  = sum W[co,ci,a,b] in[ci,m+a-1,n+b-1]   (W [Cout][Cin][3][3])
 *   kind 1: conv3x3 adjoint    gin[ci,m,n]  = sum W[co,ci,a,b] g[co,m-a+1,n-b+1]
 *   kind 2: down 2x2/s2        out[co,i,j]  = sum Wd[co,ci,a,b] in[ci,2i+a,2j+b]    (Wd [Cout][Cin][2][2])
 *   kind 3: down adjoint       gin[ci,2i+a,2j+b] = sum_co Wd[co,ci,a,b] g[co,i,j]
 *   kind 4: up 2x2/s2 (transp) out[co,2i+a,2j+b] = sum_ci Wu[ci,co,a,b] in[ci,i,j]  (Wu [Cin][Cout][2][2])
 *   kind 5: up adjoint         gin[ci,i,j]  = sum Wu[ci,co,a,b] g[co,2i+a,2j+b]
 * w: HOST fp32 tensor of the conv in the layouts above, shape (s0, s1, kh, kw).
 * in/out/aux: DEVICE NHWC tensors of fp32 (precision 0) or bf16 (precision 1).
 *   Hin, Win: spatial size of `in`; out has the kind's output size.
 * epi: 0 store, 1 softplus, 2 out = acc + aux, 3 out = acc * (1 - exp(-aux)).
 * use_tc: 1 = tcgen05 kernel (precision 1: bf16 operands; precision 0: 3xTF32), 0 = FFMA kernel.
 * Synchronises the device; returns an ideq_status code.
 *
 * ideq_debug_rb runs ONE fused level-0 residual block (rbf.cu), bf16, 32 channels, W in {128, 256}:
 *   vjp 0: act = sp(A x) (written), out = x + B act
 *   vjp 1: out = x + A^T((B^T x) . (1 - exp(-act)))          (act read: the saved activation)
 * with A, B the block's two 3x3 convolutions (wA, wB: HOST fp32 [32][32][3][3]); x, out, act:
 * DEVICE NHWC bf16 [N][H][W][32].
 *
 * ideq_debug_set_fusion switches the fused residual blocks of a context's network on (1, the
 * default) or off (0: two launches per block) for the programs built afterwards (tests compare
 * the two).
 */
#ifndef IDEQ_DEBUG_H
#define IDEQ_DEBUG_H
#include "ideq.h"
#ifdef __cplusplus
extern "C" {
#endif

IDEQ_API int ideq_debug_conv(int kind, int precision, int use_tc, const float* w, int s0, int s1, int N, int Hin,
                             int Win, const void* in, void* out, const void* aux, int epi, char* err, int errlen);
IDEQ_API int ideq_debug_rb(int vjp, const float* wA, const float* wB, int N, int H, int W, const void* x, void* out,
                           void* act, char* err, int errlen);
IDEQ_API int ideq_debug_set_fusion(ideq_ctx* ctx, int on);

#ifdef __cplusplus
}
#endif
#endif
