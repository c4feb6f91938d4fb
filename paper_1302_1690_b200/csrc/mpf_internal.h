// mpf_internal.h — internal declarations of libmpf (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/mpf.h"

namespace mpf {

constexpr int kMaxL = MPF_MAX_LAYERS;

// One activation a[l] in the padded uniform-fragment layout.
//   F      fragments per image
//   vr,vc  valid rows/cols per fragment (logical size)
//   gr,gc  storage grid per fragment (row pitch gc*C floats).  A CONV/FC output is
//          stored in its *input's* grid (gr,gc of the input): positions past the valid
//          region are padding ("garbage" in forward, always zero in delta buffers).
//          Pooled outputs are compact (gr == vr).
//   C      channels (innermost)
struct Act {
  int F = 1, vr = 0, vc = 0, gr = 0, gc = 0, C = 0;
  long long elems_per_image() const { return (long long)F * gr * gc * C; }
};

enum class Where : int { None = 0, Tape = 1, ScratchY = 2 };

struct LayerPlan {
  mpf_layer L{};
  int cin = 0, cout = 0;          // channels in / out
  long long w_off = -1, b_off = -1; // canonical param offsets
  long long wpack_off = -1;       // fwd pack [co][k][k][ci]  (floats, scratch)
  long long dpack_off = -1;       // dgrad pack [ci][k][k][co] rotated
  Where out_where = Where::None;  // where a[l+1] lives
  long long tape_val_off = -1;    // bytes in tape (values)   (n_cap images)
  long long tape_idx_off = -1;    // bytes in tape (argmax, POOL)
};

// live kernel timing (mpf_profile_begin/end)
struct ProfRec {
  std::string name;
  int layer;
  double flops, bytes;
  int e0, e1;
};
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> ev;
  int used = 0;
  std::vector<ProfRec> recs;
};

// peer-memory gradient exchange (exchange.cu): byte layout of one rank's buffer
struct ExLayout {
  static constexpr size_t kEpoch = 0, kSgdCnt = 8, kTimeout = 12, kPushCnt = 256, kPeers = 512, kFlags = 1024;
  static constexpr int kMaxWorld = 64;
  int world = 1, nbmax = 1;
  long long n_params = 0;
  size_t slots = 0, bytes = 0;
};

struct Net {
  mpf_config cfg{};
  Prof prof;
  int n_layers = 0;
  LayerPlan lp[kMaxL];
  Act a[kMaxL + 1];
  int n_levels = 0, S = 1, classes = 0;
  int O_H = 0, O_W = 0, Hp = 0, Wp = 0;
  int pool_k[kMaxL];  // pool factors in order (levels)
  long long n_params = 0;
  // memory plan for n_cap images (bytes)
  int n_cap = 0;
  size_t tape_bytes = 0, scratch_bytes = 0;
  size_t y_floats = 0;  // scratch Y capacity (floats)
  size_t off_Y = 0, off_dA = 0, off_dB = 0, off_dC = 0, off_bpart = 0, off_wpack = 0, off_part = 0,
         off_nlab = 0, off_lossp = 0, off_err = 0, off_stage_img = 0, off_stage_lab = 0,
         off_stage_loss = 0, off_theta0 = 0, off_armijo = 0, off_labfrag = 0;
  // partial_reduce scratch: [0] main stream (bias / head), [1] side stream (weight gradients)
  size_t off_red[2] = {0, 0};
  size_t off_lossred = 0;  // loss_finalize chunk sums + per-image counters
  size_t off_z = 0;        // softmax FC logits [n][head positions][classes] (forward -> head)
  bool z_ready = false;    // the last forward wrote off_z
  int red_E = 0;  // widest reduction (floats per row)
  size_t stage_bytes = 0;  // one of the two host-input staging slots (images | labels)
  // host-buffer steps: inputs of step i + 1 are copied on copy_stream into the other
  // staging slot while step i computes (events order the slots' reuse)
  cudaStream_t copy_stream = nullptr;
  // backward: weight gradients run on side_stream, overlapping the dgrad / MPF-backward chain
  cudaStream_t side_stream = nullptr;
  cudaEvent_t ev_ready = nullptr, ev_join = nullptr, ev_buf[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t ev_copied[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  int stage_slot = 0;
  // data-parallel gradient buckets (mpf_net_set_grad_hook)
  mpf_grad_ready_fn grad_hook = nullptr;
  void* grad_hook_user = nullptr;
  // peer-memory gradient exchange (mpf_exchange_attach)
  bool ex_on = false, ex_in_bwd = true;
  int ex_rank = 0;
  char* ex_own = nullptr;
  ExLayout ex_layout;
  size_t part_floats = 0;  // capacity of the wgrad partial buffer (floats)
  size_t bpart_floats = 0; // capacity of the bias / head partial buffer (floats)
  int loss_parts = 0;      // loss partials per image
  // bound memory
  float* params = nullptr;
  float* grads = nullptr;
  char* tape = nullptr;
  char* scratch = nullptr;
  bool bound = false;
  // state of the last forward
  const float* images = nullptr;
  int n_fwd = 0;
  bool have_fwd = false;
};

// ---------------------------------------------------------------- kernels (launchers)
// All launchers enqueue on `s` and return cudaGetLastError().

struct ConvArgs {
  // input
  const float* in;
  int in_F;              // fragments per image of the input (grid z = n*in_F)
  int in_gr, in_gc;      // input storage grid
  int in_vr, in_vc;      // readable region (elements outside read as 0)
  int image_mode;        // 1: input is the raw image [n][Cin][H][W] (NCHW), grid (in_gr,in_gc) = (H,W)
  int off_y, off_x;      // input coordinate of output (0,0) tap (0,0): in(y+off_y+ky, x+off_x+kx)
  int cin;
  // weights [cout][k][k][cin] and bias (nullable)
  const float* w;
  const float* bias;
  int k, cout;
  // output
  float* out;
  int out_gr, out_gc;    // output storage grid (covered fully)
  int out_vr, out_vc;    // valid region; positions outside are written as 0 when zero_pad
  int act;               // activation applied in the epilogue
  const float* mul_dact; // nullable: multiply by act'(mul_dact[out position]) (deltas)
  int dact;              // activation whose derivative is applied with mul_dact
  int zero_pad;
  int round_tf32;
  int n_frag_total;      // n * in_F
};
cudaError_t launch_conv_simt(const ConvArgs& a, cudaStream_t s);

struct WgradArgs {
  const float* x;        // layer input
  int image_mode;        // x is the raw image (NCHW, zero outside H,W)
  int x_gr, x_gc, x_vr, x_vc;
  const float* dy;       // delta at pre-activation of the layer output, grid (y_gr, y_gc)
  int y_gr, y_gc, y_vr, y_vc;
  int n_frag_total;
  int cin, cout, k;
  float* part_w;         // [n_split][cout][k*k*cin]
  float* part_b;         // [n_split][cout]
  int n_split;
};
cudaError_t launch_wgrad_simt(const WgradArgs& a, cudaStream_t s);
int wgrad_simt_splits(long long positions);

// grads_canon[w_off + ((co*cin+ci)*k+ky)*k+kx] += sum_s part_w[s][co][(ky*k+kx)*cin+ci]; bias likewise.
cudaError_t launch_wgrad_reduce(const float* part_w, int n_split, int cout, int cin, int k, float* gw,
                                cudaStream_t s);

struct MpfArgs {
  const float* y;        // conv output, grid (gr,gc), valid vr x vc, C channels
  int gr, gc, vr, vc, C, k;
  int n_frag_in;         // n * F_in
  float* out;            // pooled [n*F_in*k*k][m][m][C], m = (vr-k+1)/k (uniform)
  uint8_t* idx;          // argmax dy*k+dx
  int m_r, m_c;
  int round_tf32;
};
cudaError_t launch_mpf_fwd(const MpfArgs& a, cudaStream_t s);

struct MpfBwdArgs {
  const float* dout;     // delta of the pooled output [n*F_in*k*k][m][m][C]
  const float* pooled;   // pooled values (for act')
  const uint8_t* idx;
  int gr, gc, vr, vc, C, k, m_r, m_c;
  int n_frag_in;
  int act;               // activation of the conv that produced y
  float* din;            // delta at pre-activation of y, grid (gr,gc); zero outside valid
  int round_tf32;
  float* bias_part;      // nullable: [mpf_bwd_partials(a)][C] per-block sums of din (bias gradient)
  int premul;            // 1: dout already carries act'(y) (the producing dgrad applied it); pooled unused
  int block_form;        // k = 2: one 2 x 2 block per work item instead of a band (MPF_FLAG_MPF_BWD_BLOCK)
  int scatter_form;      // k = 3: the shared-memory scatter instead of the gather (MPF_FLAG_MPF_BWD_SCATTER)
};
cudaError_t launch_mpf_bwd(const MpfBwdArgs& a, cudaStream_t s);
long long mpf_bwd_partials(const MpfBwdArgs& a);

// per-channel partial sums of a [P][C] tensor: part[channel_partials(P)][C]
long long channel_partials(long long P);
cudaError_t launch_channel_partial(const float* dy, long long P, int C, float* part, cudaStream_t s);
// dst[e] += sum_b part[b][e] for e < split_at, dst2[e - split_at] += ... beyond (fixed order).
// Scratch of this two-level reduction: up to kReduceSegments x E segment sums and one
// arrival counter per 32-column chunk (zero between launches); one scratch per stream.
constexpr int kReduceSegments = 128;
struct ReduceScratch {
  float* tmp;
  size_t tmp_floats;
  unsigned* cnt;
  int n_cnt;
};
cudaError_t launch_partial_reduce(const float* part, int nb, int E, float* dst, float* dst2, int split_at,
                                  const ReduceScratch& rs, cudaStream_t s);

struct HeadArgs {
  const float* h;        // last hidden activation, grid (gr,gc), valid (vr,vc), Ch channels
  int gr, gc, vr, vc, Ch, F; // F fragments per image
  const float* w;        // softmax FC weights canonical [C][Ch] (1x1)
  const float* b;        // [C]
  int C;
  int hidden_act;        // activation of h (for act')
  const uint8_t* labels; // [n][O_H][O_W] (training)
  int O_H, O_W;
  int n_levels;
  int pool_k[kMaxL];
  const int* nlab;       // [n]
  float cw[16];          // class weights
  float* probs;          // forward-only mode when non-null: [n*F][vr][vc][C] compact
  float* dh;             // training: [n*F][gr][gc][Ch] delta of the previous layer (zero off-valid)
  float* loss_part;      // training: [n][tiles_per_img][head_loss_parts_per_tile()]
  float* part;           // training: [n_blocks][C*Ch + C + Ch] (dW_L, db_L, db_prev)
  int tiles_per_img, n_blocks;
  int* err;
  int n;
  int round_tf32;
  const uint8_t* lab_frag;  // training: labels in head-position order (launch_label_frag), or NULL
  const float* zpre;        // logits without bias [n][F*gr*gc][C] from the last hidden layer's
                            // forward epilogue, or NULL (the head computes them from h)
};
int head_tiles_per_image(long long per_img);
// labels gathered into head-position (fragment-major) order: out[img][pos] = class, 255
// (ignored / outside the output grid) or kLabFragPad (padding of the fragment grid)
constexpr int kLabFragPad = 254;
cudaError_t launch_label_frag(const HeadArgs& a, uint8_t* out, cudaStream_t s);
int head_loss_parts_per_tile();
int head_blocks(long long total_tiles);
bool head_supported(int C, int Ch);
cudaError_t launch_head2(const HeadArgs& a, cudaStream_t s);
cudaError_t launch_label_count(const uint8_t* labels, int n, int hw, int classes, int* nlab, cudaStream_t s);
cudaError_t launch_sqnorm(const float* g, long long n, double* part, int nb, double* out, cudaStream_t s);
cudaError_t launch_armijo_axpy(float* theta, const float* theta0, const float* g, long long n, float step,
                               cudaStream_t s);
cudaError_t launch_lbfgs_gset(float* gprev, const float* g, long long n, float scale, cudaStream_t s);
cudaError_t launch_lbfgs_pair(float* S, float* Y, float* gprev, const float* theta, const float* theta0, const float* g,
                              long long n, float scale, double* part, int nb, cudaStream_t s);
cudaError_t launch_lbfgs_pass(double* v, const float* x, const float* z, long long n, const double* part_in, int mode,
                              double rho, double* a_slot, double post, double* part_out, int nb, cudaStream_t s);
cudaError_t launch_lbfgs_trial(float* theta, const float* theta0, const double* v, long long n, double alpha,
                               cudaStream_t s);
cudaError_t launch_mirror_pad(const float* in, float* out, long long planes, int H, int W, int pt, int pl, int Hp, int Wp,
                              cudaStream_t s);
cudaError_t launch_class_hist(const uint8_t* labels, long long total, int classes, unsigned long long* counts,
                              cudaStream_t s);
// loss_finalize scratch: kLossChunks x n chunk sums + n arrival counters (zero between launches)
constexpr int kLossChunks = 32;
cudaError_t launch_loss_finalize(const float* loss_part, int parts, const int* nlab, int n, float* loss, float* tmp,
                                 unsigned* cnt, cudaStream_t s);
cudaError_t launch_sgd(float* params, float* grads, long long n, float lr, float scale, cudaStream_t s);

// peer-memory gradient exchange (exchange.cu)
ExLayout exchange_layout(int world, int nbmax, long long n_params);
// copy grads[off, off+count) into this rank's slot (parity of the coming epoch) of every
// rank's buffer, then raise flag (rank, bucket) = epoch in every buffer
cudaError_t launch_exchange_push(const float* grads, long long off, long long count, char* own, const ExLayout& L,
                                 int rank, int bucket, cudaStream_t s);
// wait for every rank's flags 0 .. nb-1, theta -= lr*scale*sum_r slot[r] (rank order), g = 0, epoch++
cudaError_t launch_exchange_sgd(float* params, float* grads, float lr, float scale, char* own, const ExLayout& L,
                                int nb, cudaStream_t s);
cudaError_t launch_pack_weights(const float* w_canon, int cout, int cin, int k, float* wpack, float* dpack,
                                int round_fwd, int round_dgrad, cudaStream_t s);
cudaError_t launch_frag2pix(const float* frag, float* pix, int n, int C, int F, int fr, int fc, int O_H,
                            int O_W, int n_levels, const int* pool_k, cudaStream_t s);
cudaError_t launch_compact_copy(const float* src, int gr, int gc, int vr, int vc, int C, long long nf,
                                float* dst, cudaStream_t s);

// First layer (one input map, the raw image [n][H][W]) on CUDA cores, fp32.
struct FirstConvArgs {
  const float* img;
  int n, H, W;
  const float* w;        // canonical W[co][0][ky][kx]
  const float* bias;
  int k, cout;
  float* out;            // [n][out_gr][out_gc][cout]
  int out_gr, out_gc, out_vr, out_vc;
  int act, zero_pad, round_tf32;
  int n_cog;             // set by the launcher
};
struct FirstWgradArgs {
  const float* img;
  int n, H, W;
  const float* dy;       // [n][gr][gc][cout], zero outside the valid region
  int gr, gc;
  int k, cout;
  float* part;           // [n_blocks][cout][k*k]
  int n_blocks;
  int n_cog;             // set by the launcher
};
bool first_conv_supported(int cin, int cout, int k);
// first conv + activation + the MPF layer after it in one kernel (conv output never stored)
bool first_conv_mpf_supported(int cout, int k, int pool_k);
struct MpfArgs;
cudaError_t launch_first_conv_mpf(const FirstConvArgs& a, const MpfArgs& m, cudaStream_t s);
int first_wgrad_blocks(int k);  // k = 0: the largest grid (partial-buffer sizing)
cudaError_t launch_first_conv(FirstConvArgs a, cudaStream_t s);
cudaError_t launch_first_wgrad(FirstWgradArgs a, cudaStream_t s);

// thread-local error text
void set_error(const std::string& msg);

}  // namespace mpf

struct mpf_net : public mpf::Net {};
