/*
 * mpf.h — C ABI of libmpf: single-pass whole-image training of MaxPooling
 * Convolutional Networks with MaxPoolingFragment (MPF) layers on B200 (sm_100a).
 *
 * Method: arxiv 1302.1690.  "processes each training image in a single
 * pass": a whole image is forward-propagated through C, MPF and FC
 * layers into an output image x_hat whose every pixel equals the net applied to
 * the patch at that pixel (§3.2); the loss derivative w.r.t. x_hat
 * is back-propagated through MPF layers (Alg. 4) and through C/FC
 * layers over all fragments, summing parameter gradients over fragments (Alg. 2,
 * PAPER.md:131-140); weights are updated by SGD.
 *
 * Conventions (all calls):
 *   - Every call returns mpf_status; nothing throws or aborts across the ABI.  On a
 *     non-OK status mpf_last_error() returns a thread-local message.
 *   - Device pointers ("d_") are CUDA global-memory pointers owned by the caller
 *     (typically torch tensors).  Host pointers ("h_") are ordinary host memory;
 *     pinned memory makes the host copies asynchronous.
 *   - `stream` is a cudaStream_t passed as void*.  Every device call is enqueued on
 *     it and returns without synchronising (except mpf_check and the host-buffer
 *     step, which document their syncs).
 *   - The net owns only host metadata.  All device memory (parameters, gradients,
 *     tape, scratch) is allocated by the caller with the sizes mpf_net_memory
 *     reports and attached with mpf_net_bind.
 *   - Layout of every activation on the device is fragment-major NHWC fp32
 *     [n_images * F_l, rows, cols, C_l], fragment index
 *     f_l = f_{l-1} * k^2 + (r * k + c) with the image outermost (reading R2).
 *   - Parameters/gradients are one flat fp32 vector in the canonical order of
 *     layer order; W[out][in][kr][kc] row-major, then b[out].
 */
#ifndef MPF_H
#define MPF_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MPF_VERSION 1
#define MPF_MAX_LAYERS 24

typedef enum {
  MPF_OK = 0,
  MPF_ERR_ARG = 1,      /* NULL / out-of-range argument */
  MPF_ERR_CONFIG = 2,   /* invalid architecture or geometry */
  MPF_ERR_DATA = 3,     /* bad labels (>= classes and != 255) or image count */
  MPF_ERR_INTERNAL = 4, /* consistency failure */
  MPF_ERR_CUDA = 5,     /* a CUDA runtime/driver call failed */
  MPF_ERR_STATE = 6     /* call order violated (e.g. backward before forward, unbound net) */
} mpf_status;

/* layer kinds (§2) */
enum { MPF_CONV = 0, MPF_POOL = 1, MPF_FC = 2 };
/* activations ("tanh or logistic"); the last FC must be MPF_IDENTITY (softmax head) */
enum { MPF_TANH = 0, MPF_IDENTITY = 1, MPF_LOGISTIC = 2 };
/* precision of the tensor-core convolutions */
enum { MPF_PREC_TF32 = 0, /* TF32 operands rounded to nearest, fp32 accumulate (north_star) */
       MPF_PREC_FP32 = 1  /* fp32 CUDA-core convolutions everywhere (reference mode, slow) */ };

/*
 * One layer.  CONV: k x k valid cross-correlation with n_out maps, full connectivity
 * (PAPER.md:197), + bias, + act.  POOL: k x k max pooling, realised as an MPF layer
 * (Alg. 3; n_out, act ignored).  FC: fully-connected over the k x k x C volume left at
 * that depth in patch mode (k = 1 after the first FC), evaluated over fragments as a
 * k x k convolution (north_star; reading R12).
 */
typedef struct {
  int32_t kind, k, n_out, act;
} mpf_layer;

typedef struct {
  int32_t in_channels;  /* maps of the input image (1 for the BASELINE configs) */
  int32_t patch;        /* P: square patch = receptive field; must reduce to 1x1 exactly */
  int32_t image_rows;   /* H */
  int32_t image_cols;   /* W */
  int32_t max_images;   /* largest n passed to forward/backward */
  int32_t precision;    /* MPF_PREC_* */
  uint32_t flags;       /* MPF_FLAG_* kernel-selection flags; 0 = the measured defaults */
  int32_t debug_keep;   /* 1: keep every conv output on the tape (mpf_debug_tape), for parity tests */
} mpf_config;

/*
 * Kernel-selection flags (mpf_config.flags; changeable later with mpf_net_set_flags).  The
 * default (0) is the configuration DESIGN.md §5 measured fastest; every flag selects an
 * alternative that computes the same sums (bitwise, or to fp32 summation order where the
 * tile shape changes the order; parity-tested), for A/B measurements and tests:
 *   SERIAL      one stream: the weight packs and weight gradients do not overlap the main
 *               chain on the side stream (results bitwise identical: fixed-order reductions).
 *   TC_SINGLE   tensor-core convolutions and weight gradients without CTA pairs (M = 128 per CTA).
 *   TC_PAIR     CTA pairs (cta_group::2, M = 256) wherever they fit.
 *   NTAP_ON     the multi-tap convolution on every eligible narrow layer (default: k >= 5).
 *   NTAP_OFF    never the multi-tap convolution.
 *   NTAP_NO_MC  no cluster multicast: neither the multi-tap convolution's weights nor the
 *               weight gradients' dY tile (bitwise identical results).
 *   WGRAD_M128  C_out <= 64 weight gradients with C_out on M (M = 128 tiles) instead of the
 *               default swapped roles (M = 128 rows of (tap, input channel), N = C_out).
 *   ROLE_TIMERS per-warp-role cycle counters of the tensor-core convolutions printed to
 *               stderr after every launch (synchronises; profiling only).
 *   FUSE_FIRST_POOL  the first conv + activation + the MPF layer after it in one kernel
 *               (the conv output never reaches device memory; bitwise equal).
 *   HEAD_LOGITS_OFF  the softmax FC's logits are computed by the head kernel from h instead
 *               of in the epilogue of the last hidden layer's tensor-core forward (same sums
 *               to fp32 summation order).  Default: in the epilogue when that layer's
 *               k^2 C_in >= 512.
 *   HEAD_LOGITS_ON   in the epilogue whenever the last hidden layer runs on the tensor cores.
 *   MPF_BWD_BLOCK  the k = 2 MPF backward as one 2 x 2 block per work item instead of bands of
 *               block rows (bitwise the same deltas).
 *   MPF_BWD_SCATTER the k = 3 MPF backward as a shared-memory scatter (each window adds its
 *               delta to its argmax element) instead of the register-blocked gather (each
 *               element tests its k^2 candidate windows); the same sums in another fp32
 *               order.  Faster alone, slower in the overlapped step.
 */
enum {
  MPF_FLAG_SERIAL = 1u << 0,
  MPF_FLAG_TC_SINGLE = 1u << 1,
  MPF_FLAG_TC_PAIR = 1u << 2,
  MPF_FLAG_NTAP_ON = 1u << 3,
  MPF_FLAG_NTAP_OFF = 1u << 4,
  MPF_FLAG_NTAP_NO_MC = 1u << 5,
  MPF_FLAG_WGRAD_M128 = 1u << 6,
  MPF_FLAG_ROLE_TIMERS = 1u << 7,
  MPF_FLAG_FUSE_FIRST_POOL = 1u << 8,
  MPF_FLAG_HEAD_LOGITS_OFF = 1u << 9,
  MPF_FLAG_HEAD_LOGITS_ON = 1u << 10,
  MPF_FLAG_MPF_BWD_BLOCK = 1u << 11,
  MPF_FLAG_MPF_BWD_SCATTER = 1u << 12
};

/* Geometry of the padded uniform-fragment layout.
 * Activation l = 0..n_layers (a[0] = zero-padded image, a[l+1] = output of layer l). */
typedef struct {
  int32_t n_layers, n_levels, classes;
  int32_t stride;                 /* S = prod of pooling factors */
  int32_t n_fragments;            /* fragments per image at the output */
  int32_t out_rows, out_cols;     /* O = H - P + 1: valid outputs (R7) */
  int32_t padded_rows, padded_cols; /* H' = P - 1 + S * ceil(O / S) */
  int32_t frag_rows, frag_cols;   /* output grid per fragment (S * frag_rows >= out_rows) */
  int64_t n_params;
  int32_t frag[MPF_MAX_LAYERS + 1]; /* fragments per image of a[l] */
  int32_t rows[MPF_MAX_LAYERS + 1]; /* valid rows of a[l] per fragment */
  int32_t cols[MPF_MAX_LAYERS + 1];
  int32_t chans[MPF_MAX_LAYERS + 1];
  int64_t w_offset[MPF_MAX_LAYERS]; /* offset of W of layer l in the flat params, -1 for POOL */
  int64_t b_offset[MPF_MAX_LAYERS];
} mpf_geometry;

typedef struct mpf_net mpf_net; /* opaque */

/* Library version (MPF_VERSION). */
int32_t mpf_version(void);

/* Thread-local description of the last error (never NULL). */
const char* mpf_last_error(void);

/*
 * validate_arch + plan_geometry (with valid outputs instead of
 * mirror padding): checks that P reduces to 1x1 exactly at the last layer, that the
 * last layer is an FC with identity activation, and plans the padded layout.  No
 * device memory is touched.  MPF_ERR_CONFIG on an invalid architecture.
 */
mpf_status mpf_net_create(const mpf_config* cfg, const mpf_layer* layers, int32_t n_layers,
                          mpf_net** out);
void mpf_net_destroy(mpf_net* net);

mpf_status mpf_net_geometry(const mpf_net* net, mpf_geometry* out);

/* Replace the net's MPF_FLAG_* flags (takes effect at the next call that launches work).
 * MPF_ERR_ARG for unknown bits or for NTAP_ON with NTAP_OFF / TC_PAIR with TC_SINGLE. */
mpf_status mpf_net_set_flags(mpf_net* net, uint32_t flags);

/*
 * Device bytes the caller must provide for n_images images (n_images <= max_images):
 * params and grads (n_params fp32 each), the tape (pooled fragments + argmax +
 * FC activations kept from forward to backward) and scratch (transient conv
 * outputs, deltas, packed weights, reduction partials, staging for host inputs).
 * Every buffer must be 256-byte aligned (torch allocations are).
 */
mpf_status mpf_net_memory(const mpf_net* net, int32_t n_images, uint64_t* params_bytes,
                          uint64_t* grads_bytes, uint64_t* tape_bytes, uint64_t* scratch_bytes);

/* Attach caller-owned device buffers sized by mpf_net_memory(net, n_images, ...). */
mpf_status mpf_net_bind(mpf_net* net, void* d_params, void* d_grads, void* d_tape, void* d_scratch,
                        int32_t n_images);

/*
 * Whole-image forward (Alg. 1 per layer, Alg. 3 for MPF) of n images
 * d_images [n, in_channels, H, W] fp32 (read again by mpf_backward_image: keep it
 * alive and unchanged until then).  The image is zero-padded to H' x W' on the fly
 * (padded outputs are ignored by the loss).  If d_probs is not NULL, the softmax
 * output of every fragment position is written to d_probs
 * [n * n_fragments, frag_rows, frag_cols, classes] (use mpf_fragments_to_pixels to
 * reassemble x_hat).  Overwrites the tape.
 */
mpf_status mpf_forward_image(mpf_net* net, const float* d_images, int32_t n, float* d_probs,
                             void* stream);

/*
 * Loss and back-propagation for the images of the last forward.
 * d_labels [n, out_rows, out_cols] uint8 on the output grid (reading R7), 255 = ignore.
 * h_class_w: `classes` host floats (NULL = all 1; "MCCE per class").
 * Per image: loss = mean over labelled pixels of -w_t log p_t (R8), written to
 * d_loss[n] (device, may be NULL); gradients of that per-image mean are ADDED to the
 * bound gradient buffer (Alg. 2 accumulation; micro-batches sum).  Labels >= classes
 * other than 255 are ignored and raise a device flag reported by mpf_check.
 */
mpf_status mpf_backward_image(mpf_net* net, const uint8_t* d_labels, const float* h_class_w,
                              float* d_loss, void* stream);

/*
 * Forward + backward of n images in one call (the training step of PAPER.md:210 without
 * the update): exactly mpf_forward_image (no softmax output) followed by
 * mpf_backward_image.  Gradients are ADDED to the bound buffer; d_loss[n] (device, may be
 * NULL) receives the per-image mean losses.
 */
mpf_status mpf_train_step(mpf_net* net, const float* d_images, int32_t n, const uint8_t* d_labels,
                          const float* h_class_w, float* d_loss, void* stream);

/*
 * Armijo-safeguarded gradient step ("stochastic gradient descent safe-guarded
 * by the Armijo rule").  Computes the loss L0 and gradient
 * g = grad_scale * sum_images grad (mpf_train_step), then tries theta + alpha d, d = -g, for
 * alpha = alpha0, alpha0 beta, ... (at most max_backtracks + 1 trials, each a forward-only
 * loss evaluation: forward + the softmax head's loss, L = grad_scale * sum of the images'
 * mean losses) until L <= L0 - c alpha ||g||^2.  Accepted: the parameters move to that trial
 * point; otherwise they stay at theta.  The gradient buffer is zeroed either way.
 * h_out[5] = {L0, L_final, accepted alpha (0 if rejected), accepted (0/1), evaluations}.
 * Synchronises `stream` once per trial.  Errors: MPF_ERR_ARG for alpha0 <= 0, beta or c
 * outside (0, 1), n > 256; MPF_ERR_DATA for a non-finite L0 or ||g||.  The gradient
 * buffer is zeroed before the gradient pass, so leftover content does not enter g.
 */
mpf_status mpf_armijo_step(mpf_net* net, const float* d_images, int32_t n, const uint8_t* d_labels,
                           const float* h_class_w, float alpha0, float beta, float c, int32_t max_backtracks,
                           float grad_scale, float* h_out, void* stream);

/*
 * Full-batch L-BFGS ("We use LBFGS"; SURVEY §8(f) item 4;
 * reading R21 in DESIGN.md).  An mpf_lbfgs keeps, in a caller-owned device buffer of
 * mpf_lbfgs_state_bytes() bytes (256-byte aligned, e.g. a torch tensor; it must outlive the
 * handle), memory + 1 curvature-pair slots (s, y: fp32 [n_params] each), the base point
 * theta0 and the gradient g at it (fp32), and the direction v = H g (fp64); the handle holds
 * host bookkeeping only.  It works on the parameters and gradients bound to `net`, which
 * must outlive it.  One stream at a time; every call is asynchronous on `stream` except
 * where it says it synchronises.
 *
 * Primitives (the multi-GPU driver calls these with an all-reduce between; one GPU can call
 * mpf_lbfgs_step instead):
 *   set_gradient: g <- grad_scale * (the net's gradient buffer), the gradient at the
 *                 current parameters (the caller has zeroed, evaluated and, across ranks,
 *                 summed it).
 *   direction:    v <- H g by the two-loop recursion over the stored pairs (H0 = gamma I,
 *                 gamma = s^T y / y^T y of the newest pair), theta0 <- parameters;
 *                 *h_gtd = g^T d with d = -v; if that is not negative (or not finite) d falls
 *                 back to -g, *h_fallback = 1.  Synchronises `stream` once (or twice).
 *   trial:        parameters <- theta0 + alpha d.
 *   accept:       the net's gradient buffer holds the gradient at the current trial point:
 *                 s = theta - theta0, y = grad_scale grad - g, g <- grad_scale grad; the pair
 *                 is stored iff s^T y > 1e-10 (the oldest dropped beyond `memory`);
 *                 *h_stored = 0/1.  Synchronises `stream`.
 *   reject:       parameters <- theta0; the pairs are cleared (restart).
 *   reset:        pairs cleared and g marked unknown (after the parameters or data change).
 * Errors: MPF_ERR_ARG for memory outside [1, 64], NULL pointers, a misaligned or too small
 * state buffer; MPF_ERR_STATE for direction without a gradient, trial/accept without a
 * direction.
 */
typedef struct mpf_lbfgs mpf_lbfgs; /* opaque */
mpf_status mpf_lbfgs_state_bytes(const mpf_net* net, int32_t memory, uint64_t* bytes);
mpf_status mpf_lbfgs_create(mpf_net* net, int32_t memory, void* d_state, uint64_t state_bytes, mpf_lbfgs** out);
void mpf_lbfgs_destroy(mpf_lbfgs* lb);
mpf_status mpf_lbfgs_reset(mpf_lbfgs* lb);
mpf_status mpf_lbfgs_set_gradient(mpf_lbfgs* lb, float grad_scale, void* stream);
mpf_status mpf_lbfgs_direction(mpf_lbfgs* lb, double* h_gtd, int32_t* h_fallback, void* stream);
mpf_status mpf_lbfgs_trial(mpf_lbfgs* lb, double alpha, void* stream);
mpf_status mpf_lbfgs_accept(mpf_lbfgs* lb, float grad_scale, int32_t* h_stored, void* stream);
mpf_status mpf_lbfgs_reject(mpf_lbfgs* lb, void* stream);
/*
 * One full-batch L-BFGS iteration on one GPU over the n images (the whole training set;
 * pass the same images every call, or mpf_lbfgs_reset first): the loss and gradient at
 * theta (L = grad_scale * sum of the images' mean losses, g = grad_scale * sum of their
 * gradients; evaluated here on the first call, after mpf_lbfgs_reset, and after
 * mpf_lbfgs_set_gradient (which leaves the loss unknown); otherwise kept: from the
 * previous accepted trial, or, after a rejected search, those at the restored theta0),
 * the direction, then trials
 * theta0 + alpha d for alpha = alpha0 (empty history) or 1, times beta per backtrack, each a
 * full loss + gradient evaluation (mpf_train_step), until L <= L0 + c alpha g^T d; then
 * accept (pair update) or, after max_backtracks + 1 trials, reject.
 * h_out[7] = {L0, L_final, accepted alpha (0 if rejected), accepted (0/1), evaluations,
 * steepest-descent fallback (0/1), stored pairs}.  Synchronises once per evaluation.
 * Afterwards the gradient buffer holds the unscaled gradient of the last trial.
 * Errors: as mpf_armijo_step; MPF_ERR_DATA for a non-finite L0 or g^T d.
 */
mpf_status mpf_lbfgs_step(mpf_lbfgs* lb, const float* d_images, int32_t n, const uint8_t* d_labels,
                          const float* h_class_w, float alpha0, float beta, float c, int32_t max_backtracks,
                          float grad_scale, float* h_out, void* stream);

/*
 * The backtracking rule of the L-BFGS line search (reading
 * R21), as mpf_lbfgs_step applies it, for a caller that evaluates the (e.g. rank-summed) loss
 * itself and drives the mpf_lbfgs_* primitives (paper_1302_1690_b200.dist.lbfgs_iteration).
 * Host-only (no device, no state).
 * mpf_line_search_first: *alpha = alpha0 when no curvature pair is stored (n_pairs == 0),
 *   else 1 (the quasi-Newton step).
 * mpf_line_search_decide: after trial number trials_done (1-based) at step alpha gave loss
 *   L_trial: *decision = 1 (accept: L_trial finite and L_trial <= L0 + c * alpha * gtd),
 *   0 (try *alpha_next = beta * alpha) or -1 (max_backtracks + 1 trials failed: restore the
 *   start point).  MPF_ERR_ARG for parameters outside 0 < beta < 1, 0 < c < 1,
 *   max_backtracks >= 0, trials_done >= 1, or NULL outputs.
 */
mpf_status mpf_line_search_first(double alpha0, int32_t n_pairs, double* alpha);
mpf_status mpf_line_search_decide(double L0, double gtd, double c, double beta, double alpha, double L_trial,
                                  int32_t trials_done, int32_t max_backtracks, int32_t* decision,
                                  double* alpha_next);

/*
 * Gradient-ready hook for data-parallel training (Alg. 2's sum extended over ranks): when
 * set, mpf_backward_image / mpf_train_step call fn(user, layer, offset, count, stream) on
 * the calling host thread right after they have enqueued the weight gradient of conv/FC
 * layer `layer`.  At that point, in the order of `stream` (a cudaStream_t as void*: the
 * net's side stream, or the caller's stream under MPF_FLAG_SERIAL), the gradient entries
 * [offset, offset + count) of the bound buffer — every W and b of layers `layer` .. L not
 * yet reported — are final, so the caller can start a collective on that bucket (e.g. an
 * NCCL all-reduce ordered after `stream`) while the backward continues below.  Buckets come
 * in decreasing offset order and cover the whole buffer exactly once per backward.  Work
 * the callback enqueues on `stream` itself is joined into the caller's stream before the
 * backward returns; work on other streams is the caller's to join.  fn = NULL removes it.
 */
typedef void (*mpf_grad_ready_fn)(void* user, int32_t layer, int64_t offset, int64_t count, void* stream);
mpf_status mpf_net_set_grad_hook(mpf_net* net, mpf_grad_ready_fn fn, void* user);

/* SGD: theta <- theta - lr * grad_scale * g ; g <- 0.  While a peer-memory
 * exchange is attached (mpf_exchange_attach) this is mpf_exchange_sgd_step: g is the sum of
 * every rank's gradient. */
mpf_status mpf_sgd_step(mpf_net* net, float lr, float grad_scale, void* stream);

/*
 * Data-parallel gradient exchange over peer memory: Alg. 2's sum
 * over fragments and positions extended over the images of every rank,
 * without a separate collective.  Each rank owns one exchange buffer that every other rank
 * can address (NVLink P2P through CUDA IPC: mpf_ipc_export / mpf_ipc_open; or, on one GPU,
 * plain device pointers).  While attached:
 *   - the backward copies every gradient bucket, as soon as it is final (the points
 *     mpf_net_set_grad_hook reports, on the same stream), into this rank's slot of EVERY
 *     rank's buffer, then raises this rank's flag for that bucket in every buffer (release,
 *     system scope) — the transfer overlaps the rest of the backward;  with
 *     push_in_backward = 0 nothing is pushed by the backward and the caller calls
 *     mpf_exchange_push once after its last backward of the step (micro-batches);
 *   - mpf_exchange_sgd_step waits (acquire) until every rank's flags carry this step's
 *     epoch, sums the ranks' slots in rank order 0 .. world-1 (the same fp32 sum on every
 *     rank, so the parameters stay bitwise identical across ranks), applies
 *     theta <- theta - lr * grad_scale * sum, zeroes this rank's gradient buffer and advances
 *     the epoch.  Slots alternate between two parities by epoch, so a rank one step ahead
 *     never overwrites a slot a slower rank still reads.
 * A wait that exceeds ~10 s (a rank that never pushes) gives up, leaves theta unchanged and
 * makes mpf_check return MPF_ERR_INTERNAL.  All calls are asynchronous on `stream`.
 *
 * mpf_exchange_bytes: size of one rank's buffer for `world` ranks.  The caller allocates it
 * on the rank's device, ZERO-FILLED, before any rank attaches (e.g. torch.zeros), and
 * keeps it alive until every rank has detached.
 * mpf_exchange_attach: d_bufs[r] = rank r's buffer as addressable from this process
 * (d_bufs[rank] = the own buffer); host array of `world` pointers, copied.  MPF_ERR_ARG for
 * rank / world out of range (world <= 64) or NULL pointers; MPF_ERR_STATE if not bound.
 * mpf_exchange_detach: back to mpf_sgd_step's local update (no device work).
 */
mpf_status mpf_exchange_bytes(const mpf_net* net, int32_t world, size_t* bytes);
mpf_status mpf_exchange_attach(mpf_net* net, int32_t rank, int32_t world, void* const* d_bufs,
                               int32_t push_in_backward);
mpf_status mpf_exchange_push(mpf_net* net, void* stream);
mpf_status mpf_exchange_sgd_step(mpf_net* net, float lr, float grad_scale, void* stream);
mpf_status mpf_exchange_detach(mpf_net* net);

/*
 * CUDA IPC for the exchange buffers (legacy cudaIpc*, P2P over NVLink between the processes
 * of one node).  mpf_ipc_export: 64-byte handle of the allocation containing d_ptr (any
 * pointer into a cudaMalloc allocation, e.g. a PyTorch tensor) and d_ptr's byte offset in
 * it.  mpf_ipc_open: maps another process's allocation, *d_ptr = its base + offset.
 * mpf_ipc_close: unmaps (pass the pointer mpf_ipc_open returned).  MPF_ERR_CUDA on failure
 * (e.g. expandable-segment allocations, which cudaIpc cannot export).
 */
mpf_status mpf_ipc_export(const void* d_ptr, void* handle64, uint64_t* offset);
mpf_status mpf_ipc_open(const void* handle64, uint64_t offset, void** d_ptr);
mpf_status mpf_ipc_close(void* d_ptr, uint64_t offset);

/*
 * One end-to-end step on HOST buffers: async copy h_images [n, in_channels, H, W]
 * and h_labels [n, out_rows, out_cols] into the bound staging area, mpf_train_step,
 * and an async copy of the per-image losses to h_loss[n].  If apply_sgd,
 * also mpf_sgd_step(lr, grad_scale).  h_loss is valid after the stream is synchronised.
 * The uploads run on the net's own copy stream into one of two staging slots (ordered
 * by events against the compute on `stream`), so back-to-back calls overlap the next
 * step's upload with this step's kernels.  h_images / h_labels must stay unchanged until
 * `stream` is synchronised (pinned memory for truly asynchronous copies).
 */
mpf_status mpf_train_step_host(mpf_net* net, const float* h_images, const uint8_t* h_labels,
                               int32_t n, const float* h_class_w, float* h_loss, int32_t apply_sgd,
                               float lr, float grad_scale, void* stream);

/*
 * Defragmentation (lineage_to_pixel SPEC.md:71-79): d_frag
 * [n * n_fragments, frag_rows, frag_cols, channels] -> d_pixels [n, channels,
 * out_rows, out_cols], out(y, x) = frag[f(y, x), i(y), j(x)] with the mixed-radix
 * decode y = r1 + k1 (r2 + k2 (... + kL i)).  Padded positions are dropped.
 */
mpf_status mpf_fragments_to_pixels(const mpf_net* net, const float* d_frag, float* d_pixels,
                                   int32_t n, int32_t channels, void* stream);

/* Copy a tape tensor of the last forward (for parity tests), compact layout:
 * what = MPF_TAPE_VALUE: a[layer+1] fp32 [n*F, rows, cols, C] (POOL layers: pooled
 *        values; CONV/FC layers whose output is kept on the tape — every conv output
 *        when the net was created with debug_keep = 1)
 * what = MPF_TAPE_ARGMAX: uint8 [n*F, rows, cols, C], index dy*k + dx (POOL layers).
 * MPF_ERR_ARG if the tensor is not on the tape. */
enum { MPF_TAPE_VALUE = 0, MPF_TAPE_ARGMAX = 1 };
mpf_status mpf_debug_tape(const mpf_net* net, int32_t layer, int32_t what, void* d_dst,
                          void* stream);

/*
 * Mirror padding for same-size output ("pixels outside of the boundary of
 * testing images are synthesized by mirroring -- which allows to preserve the size of the
 * output").  d_in [planes][rows][cols] -> d_out [planes][out_rows]
 * [out_cols], pixel (yp, xp) = d_in at the reflection of (yp - pad_top, xp - pad_left) about
 * the border pixels, without repeating the edge (y < 0 -> -y, y >= rows -> 2(rows-1) - y;
 * reading R20).  For a network of patch P, pad_top = pad_left = floor((P-1)/2) and
 * out = in + P - 1 give an output grid of exactly rows x cols, output (y, x) being the patch
 * centred (R7) on pixel (y, x).  Each pad must be smaller than the image.  Async on stream.
 */
mpf_status mpf_mirror_pad(const float* d_in, int32_t planes, int32_t rows, int32_t cols, int32_t pad_top,
                          int32_t pad_left, int32_t out_rows, int32_t out_cols, float* d_out, void* stream);

/*
 * Per-class loss weights from the labels ("loss function per class because of
 * the unbalanced dataset"; the inverse-frequency rule of SURVEY §8(f) item 3):
 *     w_c = N / (C * n_c),  n_c = labelled pixels of class c in d_labels[n][out_rows][out_cols]
 *     (255 = ignored), N = sum_c n_c.
 * Counts on the device (exact integer histogram), weights on the host in double, rounded to
 * float into h_class_w[C]; optionally the counts into h_counts[C].  Synchronises `stream`.
 * Errors: MPF_ERR_DATA if a class has no labelled pixel (pass explicit weights instead).
 * The result is meant for mpf_backward_image / mpf_train_step's h_class_w.
 */
mpf_status mpf_class_weights_auto(const mpf_net* net, const uint8_t* d_labels, int32_t n, float* h_class_w,
                                  uint64_t* h_counts, void* stream);

/* Synchronise `stream` and report device-side data errors (bad labels) and CUDA errors. */
mpf_status mpf_check(mpf_net* net, void* stream);

/*
 * Live kernel timing (for bench.py's roofline): between mpf_profile_begin and
 * mpf_profile_end every kernel libmpf launches is bracketed by CUDA events recorded on
 * its own stream.  max_launches bounds the event pool (launches beyond it are not
 * timed).  mpf_profile_end synchronises the events and returns one record per
 * (kernel, layer): launch count, summed device milliseconds, and the ALGORITHMIC
 * flops and bytes of ONE launch (valid positions only, each
 * tensor read/written once, fp32 = 4 B, argmax/labels = 1 B).
 */
typedef struct {
  char name[40];
  int32_t layer;
  int32_t launches;
  double total_ms;
  double flops;  /* per launch */
  double bytes;  /* per launch */
} mpf_kernel_stat;
mpf_status mpf_profile_begin(mpf_net* net, int32_t max_launches);
mpf_status mpf_profile_end(mpf_net* net, mpf_kernel_stat* out, int32_t capacity, int32_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* MPF_H */
