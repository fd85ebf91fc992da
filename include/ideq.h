/*
 * ideq.h -- C ABI of the B200-native i-DEQ inference engine (arXiv 2605.19705).
 *
 * The library runs the inertial fixed-point iteration of the paper with frozen
 * parameters Theta = {theta, lambda, tau, alpha}:
 *
 *   z^k     = x^k + beta (x^k - x^{k-1}),   beta = 1 - alpha     PAPER Eq. 4 (l.112-114)
 *   grad  : x^{k+1} = z^k - tau (grad f(z^k, y) + lambda grad g(z^k))   Alg. 1 l.8 (l.219)
 *   prox  : x^{k+1} = prox_{tau f(., y)}(z^k - tau lambda grad g(z^k)) Alg. 2 l.7 (l.641)
 *   g(x)  = 1/2 || x - N_theta(x) ||^2,  grad g = (I - J_N)^T (x - N)  Eq. 2 (l.96-100)
 *   r_i   = ||x_i^{k+1} - x_i^k|| / ||x_i^k||, stop when r_i <= tol       l.796, l.860
 *
 * and returns x-hat = the last iterate (Remark 1, l.189-193; no averaging, no
 * restart). Everything on the iteration runs in this library's own sm_100a
 * kernels; there is no CPU fallback: without a usable B200 every call that
 * computes returns IDEQ_E_CUDA.
 *
 * Conventions
 *   - Tensors are fp32, NCHW, C-contiguous: x, y, z are [batch][C][H][W]
 *     (phase retrieval: y is [batch][J][H][W]).
 *   - "device" pointers are CUDA device memory on the context's device;
 *     "host" pointers are ordinary (preferably pinned) host memory.
 *   - The library COPIES every operator and weight buffer it is given; the
 *     caller keeps ownership of all pointers it passes.
 *   - All work is enqueued on the stream given to ideq_create. Calls that fill
 *     host outputs (ideq_solve*, stats) synchronise that stream before return.
 *   - A context is not thread-safe: one context per (process, device).
 *   - Errors: every call returns an ideq_status; a human-readable message is
 *     available from ideq_last_error(ctx). After IDEQ_E_CUDA or IDEQ_E_NCCL the
 *     context is poisoned and later calls return IDEQ_E_STATE.
 */
#ifndef IDEQ_H
#define IDEQ_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define IDEQ_ABI_VERSION 3

#if defined(__GNUC__)
#define IDEQ_API __attribute__((visibility("default")))
#else
#define IDEQ_API
#endif

typedef struct ideq_ctx ideq_ctx;

typedef enum {
  IDEQ_OK = 0,
  IDEQ_E_INVALID = 1,     /* bad shape / parameter / NULL pointer            */
  IDEQ_E_DIVERGED = 2,    /* >= 1 image produced a non-finite iterate */
  IDEQ_E_UNSUPPORTED = 3, /* e.g. PROX with PHASE: no closed form (l.1079)   */
  IDEQ_E_CUDA = 4,        /* CUDA error or no sm_100 device; ctx poisoned   */
  IDEQ_E_NCCL = 5,        /* NCCL error; ctx poisoned                        */
  IDEQ_E_NOMEM = 6,       /* device allocation failed                        */
  IDEQ_E_STATE = 7        /* ctx poisoned or call out of order               */
} ideq_status;

typedef enum {
  IDEQ_PREC_FP32 = 0, /* parity mode: fp32 storage; U-Net convolutions on tcgen05 as 3xTF32
                         (kind::tf32, hi/lo operand halves, 3 MMAs per product; widths
                         multiple of 32), the tiny net and the JFB gradient on fp32 FFMA  */
  IDEQ_PREC_BF16 = 1  /* bf16 weights/activations on tcgen05, fp32 accumulate;
                         iterate state x, z, grad g, fidelity stay fp32 (Q19) */
} ideq_precision;

typedef enum { IDEQ_NET_TINY3 = 0, IDEQ_NET_UNET4 = 1 } ideq_arch;
typedef enum { IDEQ_ACT_SOFTPLUS = 0, IDEQ_ACT_IDENTITY = 1 } ideq_act;

/*
 * Network N_theta (BASELINE.json C1 / C2 / C5; readings Q10, Q11 in DESIGN.md).
 *   TINY3: N(x) = [x +] c3(sp(c2(sp(c1(x))))), widths[0] = hidden width.
 *   UNET4: head 3x3 C->w0; per level l=0..3 res_blocks residual blocks
 *          t <- t + B(sp(A(t))); 2x2/s2 down (l<3); decoder l=2..0: 2x2/s2
 *          transposed up + additive skip, res_blocks RBs; tail 3x3 w0->C.
 *          H and W must be divisible by 8.
 *   identity_skip: 1 => N(x) = x + U(x).
 * weights: HOST fp32 blob, no biases, in this order (conv [Cout][Cin][kh][kw],
 *   transposed up [Cin][Cout][2][2]):
 *   TINY3: c1 [w][C][3][3], c2 [w][w][3][3], c3 [C][w][3][3]
 *   UNET4: head; for l=0..3: RB0.A, RB0.B, RB1.A, RB1.B, (l<3) down_l
 *          [w_{l+1}][w_l][2][2]; for l=2..0: up_l [w_{l+1}][w_l][2][2], RB0.A,
 *          RB0.B, RB1.A, RB1.B; tail [C][w0][3][3].
 * Copied at ideq_create; n_weights must match the layout exactly.
 */
typedef struct {
  ideq_arch arch;
  int channels;        /* C = 1 or 3 */
  int widths[4];
  int res_blocks;      /* UNET4: number of RBs per level (2 in all configs) */
  int identity_skip;
  ideq_act act;
  const float* weights; /* host */
  size_t n_weights;
} ideq_net_desc;

/* Data parallelism over images: rank r owns a contiguous shard. With a dist
 * descriptor (any world >= 1) the context builds an NCCL communicator and the
 * GLOBAL_MAX rule all-reduces (MAX) one float every check_every iterations; with
 * dist == NULL no NCCL call is made. nccl_id comes from ideq_get_nccl_id on rank 0
 * (the caller broadcasts it, e.g. through torch.distributed). NCCL is loaded at
 * run time (libnccl.so.2); IDEQ_E_NCCL if it is missing or a call fails. */
typedef struct {
  int rank, world;
  unsigned char nccl_id[128];
} ideq_dist;

IDEQ_API ideq_status ideq_get_nccl_id(unsigned char out[128]);

/* Create a context on `device`, enqueuing on `cuda_stream` (cudaStream_t, NULL = a stream the
 * context owns). Workspaces are sized for up to max_batch images of H x W (network activations
 * for the planned micro-batch, see ideq_create_ex; ideq_create = ideq_create_ex with opts NULL);
 * ideq_solve never allocates. dist may be NULL (single process). IDEQ_E_NOMEM when even one
 * image's workspace does not fit. */
IDEQ_API ideq_status ideq_create(const ideq_net_desc* net, ideq_precision prec, int device,
                        void* cuda_stream, int max_batch, int H, int W,
                        const ideq_dist* dist, ideq_ctx** out);

/* Workspace plan (ideq_create_ex). The solver state -- iterates, gradients, residual
 * bookkeeping -- is allocated for max_batch images; the network's activations (3 work tensors
 * per U-Net level plus the saved activation of every residual block, ~432 MB per 512 x 512 image
 * for U-Net-64 in bf16) for a MICRO-BATCH of images: a solve runs U_theta and its VJP once per
 * micro-batch, in order, then the fidelity step over the whole batch. Results do not depend on
 * the micro-batch (every kernel is per image). micro_batch = 0: the largest balanced
 * micro-batch whose workspace fits in workspace_bytes (0: 90% of the device memory left after
 * the state, minus a reserve of 2 GB + 3 planes per image for the operator and host staging).
 * With more than one micro-batch, early-stopping solves compute frozen images' tiles (the
 * live-image list indexes a whole batch). */
typedef struct {
  int micro_batch;
  size_t workspace_bytes;
} ideq_plan_opts;

IDEQ_API ideq_status ideq_create_ex(const ideq_net_desc* net, ideq_precision prec, int device,
                           void* cuda_stream, int max_batch, int H, int W,
                           const ideq_dist* dist, const ideq_plan_opts* opts, ideq_ctx** out);
/* The plan chosen at create: images per network pass and the network workspace in bytes. */
IDEQ_API ideq_status ideq_get_plan(const ideq_ctx* ctx, int* micro_batch, size_t* workspace_bytes);

typedef enum { IDEQ_OP_BLUR = 0, IDEQ_OP_INPAINT = 1, IDEQ_OP_PHASE = 2, IDEQ_OP_RICIAN = 3, IDEQ_OP_MRI = 4 } ideq_op_kind;
typedef enum { IDEQ_STEP_GRAD = 0, IDEQ_STEP_PROX = 1 } ideq_step;   /* Alg. 1 vs Alg. 2 */
typedef enum { IDEQ_BLUR_DIRECT = 0, IDEQ_BLUR_FFT = 1 } ideq_blur_impl;

/*
 * Fidelity f(x, y) (readings Q7, Q8, Q9, Q13, Q14):
 *   BLUR   : f = 1/2||k (*) x - y||^2, periodic TRUE convolution with an odd
 *            ksize kernel centred at ((ksize-1)/2, (ksize-1)/2); same kernel on
 *            every channel; grad f = A^T(Ax - y);
 *            prox = F^-1[F(v + tau A^T y) / (1 + tau |K^|^2)] (blur_impl FFT).
 *   INPAINT: f = 1/2||Mx - y||^2 (l.1009), grad = M^T(Mx - y) (l.1014),
 *            prox = (tau M y + v)/(tau M + 1) (l.1029); M shared by channels.
 *   PHASE  : f = 1/2 sum_j || |F(D_j x)|^2 - y_j ||^2, F unitary 2-D DFT,
 *            C must be 1; gradient step only.
 *   MRI    : f = 1/2||M F x - y||^2 (App. D.3.1, l.964), x real (zero phase, l.995),
 *            F the unitary 2-D DFT, y complex k-space [batch][H][W][2] (re, im),
 *            grad = Re F^-1 M (M F x - y) (l.969), prox = Re F^-1[(F v + tau M y) /
 *            (1 + tau M)] (l.985 in k-space, reading Q18); masks: HOST u8 [H][W]
 *            k-space mask shared by the batch, Hermitian-symmetric (M[-ky][-kx] =
 *            M[ky][kx], reading R7; otherwise IDEQ_E_INVALID); C = 1, power-of-two H, W.
 *   RICIAN : f = sum x^2/(2 sigma^2) - log I0(x y / sigma^2) (App. D.3.3, l.1071),
 *            grad = x/sigma^2 - (y/sigma^2) B(x y/sigma^2), B = I1/I0 (l.1075);
 *            gradient step only (no closed-form prox, l.1079); sigma > 0.
 * kernels: HOST fp32 [1 or batch][ksize][ksize]; masks: HOST u8 [batch][H][W]
 * (1 = observed); phase_masks: HOST fp32 [n_phase][H][W][2] (re, im), shared.
 * Copied; `batch` is the number of images that later solves will use: a solve with more
 * images returns IDEQ_E_INVALID.
 */
typedef struct {
  ideq_op_kind kind;
  ideq_step step;
  ideq_blur_impl blur_impl;
  int ksize, kernel_per_image;
  const float* kernels;
  const unsigned char* masks;
  int n_phase;
  const float* phase_masks;
  float sigma;  /* RICIAN noise level sigma_y > 0 */
} ideq_operator_desc;

IDEQ_API ideq_status ideq_set_operator(ideq_ctx* ctx, const ideq_operator_desc* op, int batch);

typedef enum { IDEQ_STOP_PER_IMAGE = 0, IDEQ_STOP_GLOBAL_MAX = 1 } ideq_stop_rule;

typedef struct {
  float lambda, tau, beta;   /* beta = 1 - alpha_paper in [0, 1); tau > 0; lambda >= 0 */
  int max_iter;              /* number of operator applications (reading Q2), >= 1     */
  float tol;                 /* stop when r <= tol; tol = 0 => exactly max_iter         */
  int check_every;           /* convergence checked when (k+1) % check_every == 0      */
  ideq_stop_rule stop_rule;  /* GLOBAL_MAX: max over active images (all ranks) <= tol  */
  /* Adaptive restart, Eq. 5 (l.119-121): after every accepted step k_r += 1 and
   * S += ||x^{k+1} - x^k||^2; when k_r * S > B^2 the inertia is reset (the next
   * z = x^{k+1}). restart = 0: off (the paper's inference runs without restart,
   * l.796); 1: Alg. 1 semantics (l.225: "x^{-1}, x^0 <- x^k, k <- 0", k_r and S
   * reset); 2: Alg. 2 semantics (l.647: "x^{k-1} <- x^k" only). restart_B >= 0. */
  int restart;
  float restart_B;
  /* Averaging, Alg. 1/2 steps 12-13 (l.232-237): x-hat = mean(z^0 .. z^{K0}),
   * K0 = argmin_{floor(K/2) < k < K-1} ||x^{k+1} - x^k|| (first minimum; K =
   * max_iter); empty window or diverged image -> x-hat = last accepted iterate.
   * Requires tol == 0 (fixed iteration count). 0: off (Remark 1, l.189-193). */
  int averaging;
  /* Early-stopping solves (tol > 0, PER_IMAGE) skip the network work of images that have
   * stopped: the conv kernels walk a compacted list of the active images. 0 (default): skip;
   * 1: compute every image's tiles every iteration (results are identical; for checking and
   * measurement). */
  int compute_frozen;
} ideq_params;

typedef struct {
  int iters;       /* accepted iterations; x-hat = x^{iters}                  */
  float residual;  /* last accepted r                                          */
  int status;      /* 0 converged, 1 hit max_iter, 2 diverged                  */
  int restarts;    /* number of Eq. 5 restarts                                 */
  int k0;          /* averaging: K0, or -1 when x-hat is the last iterate      */
} ideq_image_stat;

/* Solve with DEVICE y [batch][C|J][H][W] and DEVICE x_inout (in: x^0, out:
 * x-hat). stats: HOST [batch]. rmax_trace: optional HOST [max_iter] receiving
 * max_i r_i per iteration over the images active in it (NaN if none).
 * Returns IDEQ_E_DIVERGED if any image diverged (its x-hat is its last finite
 * iterate; the other images are valid). */
IDEQ_API ideq_status ideq_solve(ideq_ctx* ctx, const float* y, float* x_inout, int batch,
                       const ideq_params* p, ideq_image_stat* stats, float* rmax_trace);

/* Same, with HOST y and HOST x_inout: the host<->device copies are part of the call. */
IDEQ_API ideq_status ideq_solve_host(ideq_ctx* ctx, const float* y, float* x_inout, int batch,
                            const ideq_params* p, ideq_image_stat* stats, float* rmax_trace);

/* Component evaluations (DEVICE pointers, NCHW fp32), used for parity and by
 * callers who want the learned regularizer alone:
 *   ideq_grad_g      : grad g(z) (Eq. 2); optional u_out = N(z) - z (may be NULL)
 *   ideq_fidelity_grad: grad f(x, y)
 *   ideq_fidelity_prox: prox_{tau f(., y)}(v)                                   */
IDEQ_API ideq_status ideq_grad_g(ideq_ctx* ctx, const float* z, float* grad_out, float* u_out, int batch);
IDEQ_API ideq_status ideq_fidelity_grad(ideq_ctx* ctx, const float* y, const float* x, float* out, int batch);
IDEQ_API ideq_status ideq_fidelity_prox(ideq_ctx* ctx, const float* y, const float* v, float tau,
                               float* out, int batch);

/* JFB training gradient at the fixed point.
 * Loss L = 1/2 sum_i ||T(x_hat_i) - x*_i||^2 with ONE more i-DEQ step at x_hat treated as a
 * constant (x^{k-1} = x^k = x_hat, so z = x_hat):
 *   gradient step (Alg. 1 l.8): T = z - tau (grad f(z) + lam grad g_theta(z))
 *   prox step (Alg. 2 l.7):     T = prox_{tau f}(z - tau lam grad g_theta(z))  (inpainting only)
 * y, x_hat, x_star: DEVICE, NCHW fp32, `batch` images (the operator set by ideq_set_operator).
 * p: lambda and tau are read (beta is irrelevant at z = x_hat).
 * dtheta: HOST, n_weights floats, the blob order of ideq_create; overwritten.
 * dlam, dtau, dbeta, loss: HOST scalars (dbeta = 0 exactly).
 * Requires the fp32 context (IDEQ_PREC_FP32), identity skip and softplus (else
 * IDEQ_E_UNSUPPORTED), a prox step only with the inpainting operator. Synchronous; its tape
 * (two streams of every activation) lives in a per-context scratch pool that grows on first use
 * and is reused by later calls of the same shape (freed by ideq_destroy). */
IDEQ_API ideq_status ideq_jfb_grad(ideq_ctx* ctx, const float* y, const float* x_hat, const float* x_star,
                                   int batch, const ideq_params* p, float* dtheta, float* dlam,
                                   float* dtau, float* dbeta, float* loss);

/* Profiling: when enabled, solves launch eagerly (no CUDA graph) and bracket every
 * kernel launch with CUDA events on the context stream; ideq_get_profile returns
 * per-kernel-class totals accumulated since the last reset. */
typedef enum {
  IDEQ_K_CONV_TC = 0,     /* tcgen05 implicit-GEMM convolutions (bf16)      */
  IDEQ_K_CONV_SIMT = 1,   /* FFMA implicit-GEMM convolutions (fp32 mode)     */
  IDEQ_K_HEADTAIL = 2,    /* C <-> w0 3x3 convolutions                       */
  IDEQ_K_FIDELITY = 3,    /* blur passes, FFT passes, phase pointwise        */
  IDEQ_K_STEP = 4,        /* fused update + residual partials                 */
  IDEQ_K_REDUCE = 5,      /* per-image residual finalize + stop logic        */
  IDEQ_K_NCLASSES = 6
} ideq_kernel_class;

typedef struct {
  double ms[IDEQ_K_NCLASSES];
  long long launches[IDEQ_K_NCLASSES];
  double flops[IDEQ_K_NCLASSES];   /* algorithmic FLOPs issued by the class      */
  double bytes[IDEQ_K_NCLASSES];   /* algorithmic HBM bytes issued by the class  */
} ideq_profile;

IDEQ_API ideq_status ideq_set_profiling(ideq_ctx* ctx, int enable);
IDEQ_API ideq_status ideq_get_profile(ideq_ctx* ctx, ideq_profile* out, int reset);

/* In-graph timing of one kernel class (ideq_kernel_class: CONV_TC, CONV_SIMT, HEADTAIL, STEP --
 * with its fidelity passes -- or REDUCE) of the LAST solve's iteration: that iteration is captured
 * again into a CUDA graph (same kernels, order and launch configuration) with event-record nodes
 * wherever the class of consecutive launches changes, and replayed `reps` times; *ms = the summed
 * duration of the class's runs of launches per iteration (<= the iteration's time by
 * construction); flops / bytes = the class's algorithmic FLOPs and HBM bytes per iteration;
 * iter_ms (may be NULL) = the summed duration of every class's runs, i.e. the bracketed
 * iteration (ms / iter_ms = the class's share of an iteration). The
 * update writes into scratch: the caller's buffers are untouched, the context's solver state is
 * overwritten. IDEQ_E_STATE before the first solve. */
IDEQ_API ideq_status ideq_time_class(ideq_ctx* ctx, int kernel_class, int reps, double* ms, double* flops,
                                     double* bytes, double* iter_ms);

/* Number of kernel launches one iteration issues (for the bench's gpu_launches). */
IDEQ_API int ideq_launches_per_iteration(const ideq_ctx* ctx);

IDEQ_API const char* ideq_last_error(const ideq_ctx* ctx);
IDEQ_API void ideq_destroy(ideq_ctx* ctx);
IDEQ_API int ideq_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* IDEQ_H */
