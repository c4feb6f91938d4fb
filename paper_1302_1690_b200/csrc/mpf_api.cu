// mpf_api.cu — host side of libmpf: the C ABI declared in include/mpf.h.
//
// Geometry planning (validate_arch + plan_geometry, SPEC.md:241-258 with valid
// outputs), memory plan, and the per-step launch sequence:
//   forward  (Alg. 1 per layer, Alg. 3 for MPF)
//   loss     (MCCE per pixel, dL/dx_hat first)
//   backward (Alg. 4 for MPF, Alg. 2 accumulation)
//   SGD
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "conv_tc.h"
#include "mpf_internal.h"

namespace mpf {

static thread_local std::string g_err = "no error";
void set_error(const std::string& m) { g_err = m; }

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

#define MPF_CUDA(call)                                                                  \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess) {                                                            \
      set_error(std::string(#call) + ": " + cudaGetErrorString(_e));                    \
      return MPF_ERR_CUDA;                                                              \
    }                                                                                   \
  } while (0)

constexpr int kArmijoParts = 592;  // blocks of the deterministic ||g||^2 reduction

static mpf_status fail(mpf_status s, const std::string& m) {
  set_error(m);
  return s;
}

// ------------------------------------------------------------------ live kernel timing
static int prof_mark(Net* N, cudaStream_t s) {
  Prof& P = N->prof;
  if (!P.on || P.used + 2 > (int)P.ev.size()) return -1;
  cudaEventRecord(P.ev[P.used], s);
  return P.used++;
}
static void prof_rec(Net* N, cudaStream_t s, int e0, const char* name, int layer, double flops, double bytes) {
  Prof& P = N->prof;
  if (e0 < 0) return;
  cudaEventRecord(P.ev[P.used], s);
  P.recs.push_back(ProfRec{name, layer, flops, bytes, e0, P.used});
  P.used++;
}
// every kernel launch of the path goes through LAUNCH (timed when profiling is on)
// NVTX range per kernel launch (message = the profile name, payload = the layer), so ncu
// (--nvtx --nvtx-include) and nsys can attribute launches to layers; with no tool attached
// an NVTX call is a test of a null function pointer.
struct NvtxRange {
  NvtxRange(const char* name, int layer) {
    nvtxEventAttributes_t ea = {};
    ea.version = NVTX_VERSION;
    ea.size = NVTX_EVENT_ATTRIB_STRUCT_SIZE;
    ea.messageType = NVTX_MESSAGE_TYPE_ASCII;
    ea.message.ascii = name;
    ea.payloadType = NVTX_PAYLOAD_TYPE_INT32;
    ea.payload.iValue = layer;
    nvtxRangePushEx(&ea);
  }
  ~NvtxRange() { nvtxRangePop(); }
};

#define LAUNCH(N, s, name, layer, flops, bytes, call)            \
  do {                                                           \
    NvtxRange _nv((name), (layer));                              \
    const int _e0 = prof_mark((N), (s));                         \
    MPF_CUDA(call);                                              \
    prof_rec((N), (s), _e0, (name), (layer), (flops), (bytes));  \
  } while (0)

// ------------------------------------------------------------------ geometry plan
static mpf_status plan(Net* N) {
  const mpf_config& c = N->cfg;
  const int nl = N->n_layers;
  if (nl < 2 || nl > kMaxL) return fail(MPF_ERR_CONFIG, "n_layers must be in [2, MPF_MAX_LAYERS]");
  if (c.in_channels < 1 || c.patch < 1 || c.max_images < 1)
    return fail(MPF_ERR_CONFIG, "in_channels, patch and max_images must be >= 1");
  if (c.image_rows < c.patch || c.image_cols < c.patch)
    return fail(MPF_ERR_CONFIG, "image smaller than the patch");
  // patch-mode shape chain: exact divisibility, FC sees the whole remaining volume
  int sz = c.patch, ch = c.in_channels;
  long long off = 0;
  N->n_levels = 0;
  N->S = 1;
  for (int l = 0; l < nl; ++l) {
    const mpf_layer& L = N->lp[l].L;
    LayerPlan& P = N->lp[l];
    if (L.k < 1) return fail(MPF_ERR_CONFIG, "layer " + std::to_string(l) + ": k < 1");
    if (L.kind == MPF_POOL) {
      if (sz % L.k) return fail(MPF_ERR_CONFIG, "layer " + std::to_string(l) + ": pooling does not divide the patch-mode size");
      if (L.k > 15) return fail(MPF_ERR_CONFIG, "pool factor > 15");
      sz /= L.k;
      P.cin = P.cout = ch;
      N->pool_k[N->n_levels++] = L.k;
      N->S *= L.k;
    } else if (L.kind == MPF_CONV || L.kind == MPF_FC) {
      if (L.n_out < 1 || L.k > sz) return fail(MPF_ERR_CONFIG, "layer " + std::to_string(l) + ": bad kernel/maps");
      if (L.kind == MPF_FC && L.k != sz)
        return fail(MPF_ERR_CONFIG, "layer " + std::to_string(l) + ": FC kernel must equal the remaining spatial size");
      if (L.act != MPF_TANH && L.act != MPF_IDENTITY && L.act != MPF_LOGISTIC)
        return fail(MPF_ERR_CONFIG, "unknown activation");
      P.cin = ch;
      P.cout = L.n_out;
      P.w_off = off;
      off += (long long)L.n_out * ch * L.k * L.k;
      P.b_off = off;
      off += L.n_out;
      ch = L.n_out;
      sz = sz - L.k + 1;
    } else {
      return fail(MPF_ERR_CONFIG, "unknown layer kind");
    }
  }
  if (sz != 1) return fail(MPF_ERR_CONFIG, "the layer list does not reduce the patch to 1x1");
  const mpf_layer& last = N->lp[nl - 1].L;
  if (last.kind != MPF_FC || last.k != 1 || last.act != MPF_IDENTITY)
    return fail(MPF_ERR_CONFIG, "the last layer must be a 1x1 FC with identity activation (softmax head)");
  const mpf_layer& prev = N->lp[nl - 2].L;
  if (prev.kind == MPF_POOL) return fail(MPF_ERR_CONFIG, "the layer before the softmax FC must be CONV/FC");
  if (last.n_out > 16 || last.n_out < 2) return fail(MPF_ERR_CONFIG, "2..16 classes supported");
  if (!head_supported(last.n_out, N->lp[nl - 2].L.n_out))
    return fail(MPF_ERR_CONFIG, "the layer before the softmax FC must have <= 256 maps");
  if (N->lp[0].L.kind == MPF_POOL) return fail(MPF_ERR_CONFIG, "the first layer must be a CONV layer");
  N->classes = last.n_out;
  N->n_params = off;
  // dense geometry: valid outputs O = H - P + 1, padded so every fragment has equal size
  N->O_H = c.image_rows - c.patch + 1;
  N->O_W = c.image_cols - c.patch + 1;
  const int fr = (N->O_H + N->S - 1) / N->S, fc = (N->O_W + N->S - 1) / N->S;
  int r = fr, q = fc;
  for (int l = nl - 1; l >= 0; --l) {
    const mpf_layer& L = N->lp[l].L;
    if (L.kind == MPF_POOL) { r = r * L.k + L.k - 1; q = q * L.k + L.k - 1; }
    else { r += L.k - 1; q += L.k - 1; }
  }
  N->Hp = r;
  N->Wp = q;
  // forward chain of activations
  Act a0;
  a0.F = 1; a0.vr = a0.gr = N->Hp; a0.vc = a0.gc = N->Wp; a0.C = c.in_channels;
  N->a[0] = a0;
  for (int l = 0; l < nl; ++l) {
    const mpf_layer& L = N->lp[l].L;
    const Act& in = N->a[l];
    Act o;
    if (L.kind == MPF_POOL) {
      const int nr = in.vr - L.k + 1, nc = in.vc - L.k + 1;
      if (nr % L.k || nc % L.k) return fail(MPF_ERR_INTERNAL, "non-uniform fragments (planner bug)");
      o.F = in.F * L.k * L.k; o.vr = o.gr = nr / L.k; o.vc = o.gc = nc / L.k; o.C = in.C;
    } else {
      o.F = in.F; o.vr = in.vr - L.k + 1; o.vc = in.vc - L.k + 1; o.gr = in.gr; o.gc = in.gc; o.C = L.n_out;
    }
    if (o.vr < 1 || o.vc < 1) return fail(MPF_ERR_INTERNAL, "empty activation (planner bug)");
    N->a[l + 1] = o;
  }
  if (N->a[nl].vr != fr || N->a[nl].vc != fc) return fail(MPF_ERR_INTERNAL, "output grid mismatch (planner bug)");
  // where every layer output lives
  for (int l = 0; l < nl; ++l) {
    const mpf_layer& L = N->lp[l].L;
    if (l == nl - 1) N->lp[l].out_where = Where::None;                 // logits: fused in the head
    else if (L.kind == MPF_POOL) N->lp[l].out_where = Where::Tape;     // pooled values + argmax
    else if (N->lp[l + 1].L.kind == MPF_POOL && !c.debug_keep) N->lp[l].out_where = Where::ScratchY;  // consumed by MPF
    else N->lp[l].out_where = Where::Tape;                             // input of a CONV/FC + act'
  }
  return MPF_OK;
}

static void layout_memory(Net* N, int n) {
  size_t tape = 0;
  long long maxY = 0, maxD = 0;
  for (int l = 0; l < N->n_layers; ++l) {
    LayerPlan& P = N->lp[l];
    const Act& o = N->a[l + 1];
    const long long e = o.elems_per_image() * n;
    P.tape_val_off = P.tape_idx_off = -1;
    if (P.out_where == Where::Tape) {
      P.tape_val_off = (long long)tape;
      tape = align256(tape + sizeof(float) * e);
      if (P.L.kind == MPF_POOL) {
        P.tape_idx_off = (long long)tape;
        tape = align256(tape + e);
      }
    } else if (P.out_where == Where::ScratchY) {
      maxY = std::max(maxY, e);
    }
    if (l < N->n_layers - 1) maxD = std::max(maxD, e);
  }
  N->tape_bytes = std::max<size_t>(tape, 256);
  size_t s = 0;
  N->off_Y = s; s = align256(s + sizeof(float) * maxY);
  N->y_floats = maxY;
  N->off_dA = s; s = align256(s + sizeof(float) * maxD);
  N->off_dB = s; s = align256(s + sizeof(float) * maxD);
  N->off_dC = s; s = align256(s + sizeof(float) * maxD);  // third delta buffer (overlapped wgrads)
  // weight packs
  N->off_wpack = s;
  long long wp = 0;
  size_t max_part = 0;
  for (int l = 0; l < N->n_layers; ++l) {
    LayerPlan& P = N->lp[l];
    if (P.L.kind == MPF_POOL) continue;
    const long long nw = (long long)P.cout * P.cin * P.L.k * P.L.k;
    P.wpack_off = wp; wp += (nw + 63) / 64 * 64;
    P.dpack_off = wp; wp += (nw + 63) / 64 * 64;
    max_part = std::max<size_t>(max_part, (size_t)(nw + P.cout));
  }
  s = align256(s + sizeof(float) * wp);
  N->off_part = s;
  N->part_floats = max_part * (size_t)kMaxSplits;
  {  // the first layer's CUDA-core weight gradient writes one partial per CTA
    const LayerPlan& P0 = N->lp[0];
    N->part_floats = std::max(N->part_floats, (size_t)first_wgrad_blocks(0) * P0.cout * P0.L.k * P0.L.k);
  }
  s = align256(s + sizeof(float) * N->part_floats);
  N->off_nlab = s; s = align256(s + sizeof(int) * n);
  // bias / head partials (fixed-order two-level reductions)
  const Act& h = N->a[N->n_layers - 1];
  const long long h_pos = h.elems_per_image() / h.C;
  N->loss_parts = head_tiles_per_image(h_pos) * head_loss_parts_per_tile();
  N->off_labfrag = s; s = align256(s + (size_t)n * h_pos);  // labels in head-position order
  // the softmax FC's logits from the last hidden layer's forward epilogue, forward -> head
  N->off_z = s; s = align256(s + sizeof(float) * (size_t)n * h_pos * N->classes);
  size_t bp = (size_t)head_blocks((long long)head_tiles_per_image(h_pos) * n) *
              ((size_t)N->classes * h.C + N->classes + h.C);
  for (int l = 0; l < N->n_layers - 1; ++l) {
    const LayerPlan& P = N->lp[l];
    const Act& in = N->a[l];
    if (P.L.kind == MPF_POOL) {
      MpfBwdArgs m{};
      m.gr = in.gr; m.gc = in.gc; m.C = in.C; m.n_frag_in = n * in.F; m.k = P.L.k;
      for (int pm = 0; pm <= 1; ++pm)  // every kernel variant (premultiplied or not, band or block,
        for (int bf = 0; bf <= 1; ++bf)  // scatter or gather)
          for (int gf = 0; gf <= 1; ++gf) {
            m.premul = pm;
            m.block_form = bf;
            m.scatter_form = gf;
            bp = std::max(bp, (size_t)mpf_bwd_partials(m) * in.C);
          }
    } else {
      const Act& o = N->a[l + 1];
      bp = std::max(bp, (size_t)channel_partials((long long)n * o.F * o.gr * o.gc) * o.C);
    }
  }
  N->bpart_floats = bp;
  N->off_bpart = s; s = align256(s + sizeof(float) * bp);
  N->off_lossp = s; s = align256(s + sizeof(float) * (size_t)N->loss_parts * n);
  N->off_lossred = s; s = align256(s + (sizeof(float) * kLossChunks + sizeof(unsigned)) * (size_t)n);
  N->off_err = s; s = align256(s + 256);
  {  // two-level reduction scratch, one per stream (see launch_partial_reduce)
    const LayerPlan& P0 = N->lp[0];
    int E = N->classes * h.C + N->classes + h.C;
    E = std::max(E, P0.cout * P0.L.k * P0.L.k);
    for (int l = 0; l < N->n_layers; ++l) E = std::max(E, N->lp[l].cout);
    N->red_E = E;
    for (int r = 0; r < 2; ++r) {
      N->off_red[r] = s;
      s = align256(s + sizeof(float) * (size_t)kReduceSegments * E + sizeof(unsigned) * ((E + 31) / 32));
    }
  }
  {  // two staging slots [images | labels] for host-buffer steps
    const size_t s0 = s;
    N->off_stage_img = s; s = align256(s + sizeof(float) * (size_t)n * N->cfg.in_channels * N->cfg.image_rows * N->cfg.image_cols);
    N->off_stage_lab = s; s = align256(s + (size_t)n * N->O_H * N->O_W);
    N->stage_bytes = s - s0;
    s += N->stage_bytes;
  }
  N->off_stage_loss = s; s = align256(s + sizeof(float) * n);
  N->off_theta0 = s; s = align256(s + sizeof(float) * (size_t)N->n_params);  // Armijo: parameters at the base point
  N->off_armijo = s; s = align256(s + sizeof(double) * (kArmijoParts + 1));
  N->scratch_bytes = s;
  N->n_cap = n;
}

static float* tape_val(const Net* N, int l) { return (float*)(N->tape + N->lp[l].tape_val_off); }
static uint8_t* tape_idx(const Net* N, int l) { return (uint8_t*)(N->tape + N->lp[l].tape_idx_off); }
static float* scr(const Net* N, size_t off) { return (float*)(N->scratch + off); }
static ReduceScratch red_scratch(const Net* N, int which) {
  ReduceScratch r;
  r.tmp = scr(N, N->off_red[which]);
  r.tmp_floats = (size_t)kReduceSegments * N->red_E;
  r.cnt = (unsigned*)(r.tmp + r.tmp_floats);
  r.n_cnt = (N->red_E + 31) / 32;
  return r;
}

// pointer to activation a[l] (l >= 1) as produced in the last forward
static const float* act_ptr(const Net* N, int l) {
  const LayerPlan& P = N->lp[l - 1];
  if (P.out_where == Where::Tape) return tape_val(N, l - 1);
  if (P.out_where == Where::ScratchY) return scr(N, N->off_Y);
  return nullptr;
}

static bool use_tc(const Net* N, const LayerPlan& P, bool dgrad) {
  if (N->cfg.precision != MPF_PREC_TF32) return false;
  return tc_supported(dgrad ? P.cout : P.cin, dgrad ? P.cin : P.cout, P.L.k);
}

}  // namespace mpf

using namespace mpf;

extern "C" {

int32_t mpf_version(void) { return MPF_VERSION; }
const char* mpf_last_error(void) { return g_err.c_str(); }

mpf_status mpf_net_create(const mpf_config* cfg, const mpf_layer* layers, int32_t n_layers, mpf_net** out) {
  if (!cfg || !layers || !out) return fail(MPF_ERR_ARG, "NULL argument");
  *out = nullptr;
  if (n_layers < 2 || n_layers > kMaxL) return fail(MPF_ERR_CONFIG, "n_layers out of range");
  mpf_net* N = new mpf_net();
  N->cfg = *cfg;
  N->n_layers = n_layers;
  for (int l = 0; l < n_layers; ++l) N->lp[l].L = layers[l];
  mpf_status st = mpf_net_set_flags(N, cfg->flags);
  if (st != MPF_OK) {
    delete N;
    return st;
  }
  st = plan(N);
  if (st != MPF_OK) {
    delete N;
    return st;
  }
  layout_memory(N, cfg->max_images);
  *out = N;
  return MPF_OK;
}

void mpf_net_destroy(mpf_net* net) {
  if (!net) return;
  for (cudaEvent_t e : net->prof.ev) cudaEventDestroy(e);
  if (net->side_stream) {
    cudaStreamSynchronize(net->side_stream);
    cudaStreamDestroy(net->side_stream);
    cudaEventDestroy(net->ev_ready);
    cudaEventDestroy(net->ev_join);
    for (int i = 0; i < 3; ++i) cudaEventDestroy(net->ev_buf[i]);
  }
  if (net->copy_stream) {
    cudaStreamSynchronize(net->copy_stream);
    cudaStreamDestroy(net->copy_stream);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(net->ev_copied[i]);
      cudaEventDestroy(net->ev_free[i]);
    }
  }
  delete net;
}

mpf_status mpf_profile_begin(mpf_net* N, int32_t max_launches) {
  if (!N || max_launches < 1) return fail(MPF_ERR_ARG, "bad argument");
  Prof& P = N->prof;
  const int need = 2 * max_launches;
  while ((int)P.ev.size() < need) {
    cudaEvent_t e;
    MPF_CUDA(cudaEventCreate(&e));
    P.ev.push_back(e);
  }
  P.used = 0;
  P.recs.clear();
  P.on = true;
  return MPF_OK;
}

mpf_status mpf_profile_end(mpf_net* N, mpf_kernel_stat* out, int32_t cap, int32_t* n_out) {
  if (!N) return fail(MPF_ERR_ARG, "NULL net");
  Prof& P = N->prof;
  P.on = false;
  std::vector<mpf_kernel_stat> agg;
  for (const ProfRec& r : P.recs) {
    MPF_CUDA(cudaEventSynchronize(P.ev[r.e1]));
    float ms = 0.f;
    MPF_CUDA(cudaEventElapsedTime(&ms, P.ev[r.e0], P.ev[r.e1]));
    mpf_kernel_stat* hit = nullptr;
    for (auto& a : agg)
      if (a.layer == r.layer && strncmp(a.name, r.name.c_str(), sizeof(a.name)) == 0) hit = &a;
    if (!hit) {
      mpf_kernel_stat z;
      memset(&z, 0, sizeof(z));
      strncpy(z.name, r.name.c_str(), sizeof(z.name) - 1);
      z.layer = r.layer;
      z.flops = r.flops;
      z.bytes = r.bytes;
      agg.push_back(z);
      hit = &agg.back();
    }
    hit->launches += 1;
    hit->total_ms += ms;
  }
  if (n_out) *n_out = (int32_t)agg.size();
  if (out)
    for (int i = 0; i < (int)agg.size() && i < cap; ++i) out[i] = agg[i];
  P.recs.clear();
  P.used = 0;
  return MPF_OK;
}

mpf_status mpf_net_geometry(const mpf_net* N, mpf_geometry* g) {
  if (!N || !g) return fail(MPF_ERR_ARG, "NULL argument");
  memset(g, 0, sizeof(*g));
  g->n_layers = N->n_layers;
  g->n_levels = N->n_levels;
  g->classes = N->classes;
  g->stride = N->S;
  g->n_fragments = N->a[N->n_layers].F;
  g->out_rows = N->O_H;
  g->out_cols = N->O_W;
  g->padded_rows = N->Hp;
  g->padded_cols = N->Wp;
  g->frag_rows = N->a[N->n_layers].vr;
  g->frag_cols = N->a[N->n_layers].vc;
  g->n_params = N->n_params;
  for (int l = 0; l <= N->n_layers; ++l) {
    g->frag[l] = N->a[l].F;
    g->rows[l] = N->a[l].vr;
    g->cols[l] = N->a[l].vc;
    g->chans[l] = N->a[l].C;
  }
  for (int l = 0; l < N->n_layers; ++l) {
    g->w_offset[l] = N->lp[l].w_off;
    g->b_offset[l] = N->lp[l].b_off;
  }
  return MPF_OK;
}

mpf_status mpf_net_memory(const mpf_net* N, int32_t n, uint64_t* pb, uint64_t* gb, uint64_t* tb, uint64_t* sb) {
  if (!N) return fail(MPF_ERR_ARG, "NULL net");
  if (n < 1 || n > N->cfg.max_images) return fail(MPF_ERR_ARG, "n_images must be in [1, max_images]");
  Net tmp = *N;
  layout_memory(&tmp, n);
  if (pb) *pb = sizeof(float) * (uint64_t)N->n_params;
  if (gb) *gb = sizeof(float) * (uint64_t)N->n_params;
  if (tb) *tb = tmp.tape_bytes;
  if (sb) *sb = tmp.scratch_bytes;
  return MPF_OK;
}

mpf_status mpf_net_bind(mpf_net* N, void* p, void* g, void* t, void* s, int32_t n) {
  if (!N || !p || !g || !t || !s) return fail(MPF_ERR_ARG, "NULL buffer");
  if (n < 1 || n > N->cfg.max_images) return fail(MPF_ERR_ARG, "n_images must be in [1, max_images]");
  if (((uintptr_t)t | (uintptr_t)s) & 255) return fail(MPF_ERR_ARG, "tape/scratch must be 256-byte aligned");
  if (((uintptr_t)p | (uintptr_t)g) & 15) return fail(MPF_ERR_ARG, "params/grads must be 16-byte aligned");
  layout_memory(N, n);
  N->params = (float*)p;
  N->grads = (float*)g;
  N->tape = (char*)t;
  N->scratch = (char*)s;
  N->bound = true;
  N->have_fwd = false;
  MPF_CUDA(cudaMemset(N->scratch + N->off_err, 0, 256));
  MPF_CUDA(cudaMemset(N->scratch + N->off_lossred + sizeof(float) * kLossChunks * n, 0, sizeof(unsigned) * n));
  for (int r = 0; r < 2; ++r) {  // reduction arrival counters start (and stay) at zero
    const ReduceScratch rs = red_scratch(N, r);
    MPF_CUDA(cudaMemset(rs.cnt, 0, sizeof(unsigned) * rs.n_cnt));
  }
  return MPF_OK;
}

// The side stream (and its events) used to overlap independent work with the main chain:
// weight packs in the forward, weight gradients in the backward.  MPF_FLAG_SERIAL
// serialises everything on the caller's stream.
static cudaStream_t side_stream(Net* N, cudaStream_t s) {
  if (N->cfg.flags & MPF_FLAG_SERIAL) return s;
  if (!N->side_stream) {
    if (cudaStreamCreateWithFlags(&N->side_stream, cudaStreamNonBlocking) != cudaSuccess) return s;
    cudaEventCreateWithFlags(&N->ev_ready, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&N->ev_join, cudaEventDisableTiming);
    for (int i = 0; i < 3; ++i) cudaEventCreateWithFlags(&N->ev_buf[i], cudaEventDisableTiming);
  }
  return N->side_stream;
}

// Forward (Alg. 1 per layer, Alg. 3 for MPF) of n images on stream s.
static mpf_status forward_impl(Net* N, const float* d_images, int n, float* d_probs, cudaStream_t s) {
  float* wpack = scr(N, N->off_wpack);
  const uint32_t flags = N->cfg.flags;
  // 1. weight packs (tf32-rounded for the tensor-core path), on the side stream: the first
  // layer reads the canonical weights, so the packs overlap with it and its pool
  cudaStream_t sp = side_stream(N, s);
  if (sp != s) {
    MPF_CUDA(cudaEventRecord(N->ev_ready, s));  // parameters of this step are final
    MPF_CUDA(cudaStreamWaitEvent(sp, N->ev_ready, 0));
  }
  bool packs_joined = sp == s;
  for (int l = 0; l < N->n_layers; ++l) {
    const LayerPlan& P = N->lp[l];
    if (P.L.kind == MPF_POOL) continue;
    const double nw = (double)P.cout * P.cin * P.L.k * P.L.k;
    // tf32-round a pack only when a tensor-core kernel consumes it; CUDA-core convs use fp32
    const int rf = (l > 0 && l < N->n_layers - 1 && use_tc(N, P, false)) ? 1 : 0;
    const int rd = (l > 0 && use_tc(N, P, true)) ? 1 : 0;
    LAUNCH(N, sp, "pack_weights", l, 0.0, 12.0 * nw,
           launch_pack_weights(N->params + P.w_off, P.cout, P.cin, P.L.k, wpack + P.wpack_off,
                               wpack + P.dpack_off, rf, rd, sp));
  }
  if (sp != s) MPF_CUDA(cudaEventRecord(N->ev_join, sp));
  // 2. layers (Alg. 1; Alg. 3 for MPF)
  bool pool_done = false;  // the first layer's kernel already produced the MPF after it
  bool z_ready = false;    // the last hidden layer's epilogue wrote the logits (off_z)
  for (int l = 0; l < N->n_layers - 1; ++l) {
    const LayerPlan& P = N->lp[l];
    const Act& in = N->a[l];
    const Act& o = N->a[l + 1];
    const bool first_simt = l == 0 && first_conv_supported(N->cfg.in_channels, P.cout, P.L.k);  // canonical weights
    if (!packs_joined && P.L.kind != MPF_POOL && !first_simt) {  // the first consumer of a pack
      MPF_CUDA(cudaStreamWaitEvent(s, N->ev_join, 0));
      packs_joined = true;
    }
    // the consumer of this output rounds? (TF32 operand of a tensor-core conv)
    const bool next_tc = (l + 1 < N->n_layers - 1) && N->lp[l + 1].L.kind != MPF_POOL && use_tc(N, N->lp[l + 1], false);
    if (P.L.kind == MPF_POOL && pool_done) {  // produced by the fused first conv + MPF
      pool_done = false;
      continue;
    }
    if (P.L.kind == MPF_POOL) {
      const Act& y = in;
      MpfArgs m;
      m.y = act_ptr(N, l);
      m.gr = y.gr; m.gc = y.gc; m.vr = y.vr; m.vc = y.vc; m.C = y.C; m.k = P.L.k;
      m.n_frag_in = n * y.F;
      m.out = tape_val(N, l);
      m.idx = tape_idx(N, l);
      m.m_r = o.vr; m.m_c = o.vc;
      m.round_tf32 = (l + 1 < N->n_layers - 1 && use_tc(N, N->lp[l + 1], false)) ? 1 : 0;
      const double ein = (double)n * y.F * y.vr * y.vc * y.C, eout = (double)n * o.F * o.vr * o.vc * o.C;
      LAUNCH(N, s, "mpf_fwd", l, 0.0, 4.0 * ein + 5.0 * eout, launch_mpf_fwd(m, s));
      continue;
    }
    float* out = P.out_where == Where::Tape ? tape_val(N, l) : scr(N, N->off_Y);
    const float* x = (l == 0) ? d_images : act_ptr(N, l);
    const double pos_out = (double)n * o.F * o.vr * o.vc;
    const double cflops = 2.0 * pos_out * P.cout * P.L.k * P.L.k * P.cin;
    const double in_e = (l == 0) ? (double)n * N->cfg.in_channels * N->cfg.image_rows * N->cfg.image_cols
                                 : (double)n * in.F * in.vr * in.vc * in.C;
    const double cbytes = 4.0 * (in_e + pos_out * P.cout);
    if (first_simt) {
      FirstConvArgs f{};
      f.img = d_images; f.n = n; f.H = N->cfg.image_rows; f.W = N->cfg.image_cols;
      f.w = N->params + P.w_off; f.bias = N->params + P.b_off; f.k = P.L.k; f.cout = P.cout;
      f.out = out; f.out_gr = o.gr; f.out_gc = o.gc; f.out_vr = o.vr; f.out_vc = o.vc;
      f.act = P.L.act; f.zero_pad = P.out_where == Where::Tape ? 1 : 0; f.round_tf32 = next_tc ? 1 : 0;
      const LayerPlan& Pn = N->lp[1];
      if ((flags & MPF_FLAG_FUSE_FIRST_POOL) && P.out_where == Where::ScratchY && Pn.L.kind == MPF_POOL &&
          N->n_layers > 2 && first_conv_mpf_supported(P.cout, P.L.k, Pn.L.k)) {
        // conv + activation + MPF (layer 1) in one kernel: the conv output is never stored
        const Act& po = N->a[2];
        MpfArgs m{};
        m.y = nullptr;
        m.gr = o.gr; m.gc = o.gc; m.vr = o.vr; m.vc = o.vc; m.C = o.C; m.k = Pn.L.k;
        m.n_frag_in = n * o.F;
        m.out = tape_val(N, 1);
        m.idx = tape_idx(N, 1);
        m.m_r = po.vr; m.m_c = po.vc;
        m.round_tf32 = (2 < N->n_layers - 1 && use_tc(N, N->lp[2], false)) ? 1 : 0;
        const double eout = (double)n * po.F * po.vr * po.vc * po.C;
        LAUNCH(N, s, "conv_first_mpf", l, cflops, 4.0 * in_e + 5.0 * eout, launch_first_conv_mpf(f, m, s));
        pool_done = true;
      } else {
        LAUNCH(N, s, "conv_first_fwd", l, cflops, cbytes, launch_first_conv(f, s));
      }
    } else if (l > 0 && use_tc(N, P, false)) {
      TcConvArgs t{};
      t.x = x; t.n_frag = n * in.F; t.gr = in.gr; t.gc = in.gc; t.cin = P.cin;
      t.w = wpack + P.wpack_off; t.bias = N->params + P.b_off; t.k = P.L.k; t.cout = P.cout;
      t.out = out; t.out_vr = o.vr; t.out_vc = o.vc; t.act = P.L.act; t.shift = 0;
      t.round_out = next_tc ? 1 : 0; t.mul_dact = nullptr;
      t.zero_pad = P.out_where == Where::Tape ? 1 : 0;  // tape tensors are read whole by the TC wgrad
      t.flags = flags;
      double zflops = 0.0;
      // h feeds the softmax FC: its logits come from this epilogue when the K loop per tile is
      // long enough to hide the extra epilogue work (measured: cfg4 FC1, K = 1152: head 3.5 ->
      // 2.55 ms, forward unchanged; cfg5 FC1, K = 256: forward +0.05 ms, head -0.01 ms)
      if (l == N->n_layers - 2 && !(flags & MPF_FLAG_HEAD_LOGITS_OFF) &&
          ((flags & MPF_FLAG_HEAD_LOGITS_ON) || P.L.k * P.L.k * P.cin >= 512)) {
        t.head_w = N->params + N->lp[l + 1].w_off;
        t.head_z = scr(N, N->off_z);
        t.head_C = N->classes;
        zflops = 2.0 * pos_out * P.cout * N->classes;
        z_ready = true;
      }
      LAUNCH(N, s, "conv_fwd_tc", l, cflops + zflops, cbytes + 4.0 * pos_out * N->classes * (zflops > 0),
             launch_conv_tc(t, s));
    } else {
      ConvArgs c{};
      c.in = x;
      c.in_F = in.F;
      c.image_mode = l == 0;
      if (l == 0) {
        c.in_gr = N->cfg.image_rows; c.in_gc = N->cfg.image_cols;
        c.in_vr = N->cfg.image_rows; c.in_vc = N->cfg.image_cols;
      } else {
        c.in_gr = in.gr; c.in_gc = in.gc; c.in_vr = in.vr; c.in_vc = in.vc;
      }
      c.off_y = c.off_x = 0;
      c.cin = P.cin;
      c.w = wpack + P.wpack_off;
      c.bias = N->params + P.b_off;
      c.k = P.L.k;
      c.cout = P.cout;
      c.out = out;
      c.out_gr = o.gr; c.out_gc = o.gc; c.out_vr = o.vr; c.out_vc = o.vc;
      c.act = P.L.act;
      c.mul_dact = nullptr;
      c.dact = 0;
      c.zero_pad = P.out_where == Where::Tape ? 1 : 0;
      c.round_tf32 = next_tc ? 1 : 0;
      c.n_frag_total = n * in.F;
      LAUNCH(N, s, "conv_fwd_simt", l, cflops, cbytes, launch_conv_simt(c, s));
    }
  }
  if (!packs_joined) MPF_CUDA(cudaStreamWaitEvent(s, N->ev_join, 0));  // the backward reads the packs
  N->images = d_images;
  N->n_fwd = n;
  N->have_fwd = true;
  N->z_ready = z_ready;
  // 3. optional softmax output
  if (d_probs) {
    const int L = N->n_layers - 1;
    const Act& h = N->a[L];
    HeadArgs hd{};
    hd.h = act_ptr(N, L);
    hd.gr = h.gr; hd.gc = h.gc; hd.vr = h.vr; hd.vc = h.vc; hd.Ch = h.C; hd.F = h.F;
    hd.w = N->params + N->lp[L].w_off;
    hd.b = N->params + N->lp[L].b_off;
    hd.C = N->classes;
    hd.hidden_act = N->lp[L - 1].L.act;
    hd.probs = d_probs;
    hd.n = n;
    hd.err = (int*)(N->scratch + N->off_err);
    hd.tiles_per_img = head_tiles_per_image((long long)h.F * h.gr * h.gc);
    hd.n_blocks = head_blocks((long long)hd.tiles_per_img * n);
    hd.zpre = z_ready ? scr(N, N->off_z) : nullptr;
    const double pos = (double)n * h.F * h.vr * h.vc;
    LAUNCH(N, s, "head_probs", L, hd.zpre ? 0.0 : 2.0 * pos * h.C * N->classes,
           hd.zpre ? pos * 8.0 * N->classes : pos * (4.0 * h.C + 4.0 * N->classes), launch_head2(hd, s));
  }
  return MPF_OK;
}

mpf_status mpf_forward_image(mpf_net* N, const float* d_images, int32_t n, float* d_probs, void* stream) {
  if (!N || !d_images) return fail(MPF_ERR_ARG, "NULL argument");
  if (!N->bound) return fail(MPF_ERR_STATE, "net is not bound (mpf_net_bind)");
  if (n < 1 || n > N->n_cap) return fail(MPF_ERR_DATA, "n must be in [1, bound n_images]");
  NvtxRange nv("mpf_forward_image", n);
  return forward_impl(N, d_images, n, d_probs, (cudaStream_t)stream);
}

static mpf_status wgrad(Net* N, int l, const float* x, const float* dy, int n, cudaStream_t s) {
  const LayerPlan& P = N->lp[l];
  const Act& in = N->a[l];
  const Act& o = N->a[l + 1];
  float* part = scr(N, N->off_part);
  const long long positions = (long long)n * o.F * o.vr * o.vc;
  const double Kd = (double)P.L.k * P.L.k * P.cin;
  const double wflops = 2.0 * positions * P.cout * Kd;
  const double in_e = (l == 0) ? (double)n * N->cfg.in_channels * N->cfg.image_rows * N->cfg.image_cols
                               : (double)n * in.F * in.vr * in.vc * in.C;
  const double wbytes = 4.0 * (in_e + (double)positions * P.cout);
  if (l == 0 && first_conv_supported(N->cfg.in_channels, P.cout, P.L.k)) {
    FirstWgradArgs f{};
    f.img = x; f.n = n; f.H = N->cfg.image_rows; f.W = N->cfg.image_cols;
    f.dy = dy; f.gr = o.gr; f.gc = o.gc; f.k = P.L.k; f.cout = P.cout;
    f.part = part; f.n_blocks = first_wgrad_blocks(P.L.k);
    const int E = P.cout * P.L.k * P.L.k;
    LAUNCH(N, s, "wgrad_first", l, wflops, wbytes, launch_first_wgrad(f, s));
    LAUNCH(N, s, "wgrad_reduce", l, 0.0, 4.0 * (f.n_blocks + 1.0) * E,
           launch_partial_reduce(part, f.n_blocks, E, N->grads + P.w_off, nullptr, E, red_scratch(N, 1), s));
    return MPF_OK;
  }
  if (l > 0 && N->cfg.precision == MPF_PREC_TF32 && tc_wgrad_supported(P.cin, P.cout, P.L.k)) {
    TcWgradArgs t{};
    t.x = x; t.dy = dy; t.n_frag = n * in.F; t.gr = in.gr; t.gc = in.gc; t.vr_out = o.vr; t.vc_out = o.vc;
    t.cin = P.cin; t.cout = P.cout; t.k = P.L.k;
    t.part = part;
    t.part_cap_floats = N->part_floats;
    t.flags = N->cfg.flags;
    int splits = 0;
    LAUNCH(N, s, "wgrad_tc", l, wflops, wbytes, launch_wgrad_tc(t, &splits, s));
    const long long K = (long long)P.L.k * P.L.k * P.cin;
    LAUNCH(N, s, "wgrad_reduce", l, 0.0, 4.0 * (splits + 2.0) * (P.cout * Kd),
           launch_wgrad_reduce(part, splits, P.cout, P.cin, P.L.k, N->grads + P.w_off, s));
    return MPF_OK;
  }
  WgradArgs w{};
  w.x = x;
  w.image_mode = l == 0;
  if (l == 0) {
    w.x_gr = N->cfg.image_rows; w.x_gc = N->cfg.image_cols; w.x_vr = N->cfg.image_rows; w.x_vc = N->cfg.image_cols;
  } else {
    w.x_gr = in.gr; w.x_gc = in.gc; w.x_vr = in.vr; w.x_vc = in.vc;
  }
  w.dy = dy;
  w.y_gr = o.gr; w.y_gc = o.gc; w.y_vr = o.vr; w.y_vc = o.vc;
  w.n_frag_total = n * in.F;
  w.cin = P.cin; w.cout = P.cout; w.k = P.L.k;
  const long long K = (long long)P.L.k * P.L.k * P.cin;
  int splits = wgrad_simt_splits(positions);
  while (splits > 1 && (size_t)splits * (P.cout * K + P.cout) > N->part_floats) --splits;
  w.n_split = splits;
  w.part_w = part;
  w.part_b = part + (size_t)splits * P.cout * K;
  LAUNCH(N, s, "wgrad_simt", l, wflops, wbytes, launch_wgrad_simt(w, s));
  LAUNCH(N, s, "wgrad_reduce", l, 0.0, 4.0 * (splits + 2.0) * (P.cout * Kd),
         launch_wgrad_reduce(w.part_w, splits, P.cout, P.cin, P.L.k, N->grads + P.w_off, s));
  return MPF_OK;
}

// bias gradient of conv layer l from per-block partials [nb][C] (fixed order)
static mpf_status bias_reduce(Net* N, int l, const float* part, long long nb, cudaStream_t s) {
  const LayerPlan& P = N->lp[l];
  LAUNCH(N, s, "bias_reduce", l, 0.0, 4.0 * (double)nb * P.cout,
         launch_partial_reduce(part, (int)nb, P.cout, N->grads + P.b_off, nullptr, P.cout, red_scratch(N, 0), s));
  return MPF_OK;
}

// Backward (loss first, then Alg. 4 / Alg. 2 layer by layer).  loss_only: the head's loss
// only (Armijo trial points), no gradients.
static mpf_status backward_impl(Net* N, const uint8_t* d_labels, const float* h_class_w, float* d_loss,
                                cudaStream_t s, bool loss_only = false) {
  const int n = N->n_fwd;
  const bool tf32 = N->cfg.precision == MPF_PREC_TF32;
  const int L = N->n_layers - 1;  // the softmax FC
  int* nlab = (int*)(N->scratch + N->off_nlab);
  float* lossp = scr(N, N->off_lossp);
  float* bpart = scr(N, N->off_bpart);
  LAUNCH(N, s, "label_count", -1, 0.0, (double)n * N->O_H * N->O_W,
           launch_label_count(d_labels, n, N->O_H * N->O_W, N->classes, nlab, s));
  // head: dL/dx_hat first, dh, and the softmax FC's gradient + the
  // previous layer's bias gradient as block partials
  const Act& h = N->a[L];
  // Delta buffers rotate among three; a layer's weight gradient reads its delta on the
  // side stream while the main stream continues with the dgrad and the MPF backward
  // below it.  Before a producer overwrites a buffer, the main stream waits for the
  // weight gradient that read it (two producers later).
  float* dbuf[3] = {scr(N, N->off_dA), scr(N, N->off_dB), scr(N, N->off_dC)};
  bool pending[3] = {false, false, false};
  int ci = 0;  // dbuf[ci] holds the current delta
  float* dcur = dbuf[0];
  float* dother = dbuf[1];
  cudaStream_t sw = side_stream(N, s);
  // the next producer writes dbuf[(ci + 1) % 3]: make sure no weight gradient still reads it
  auto next_out = [&]() -> float* {
    const int b = (ci + 1) % 3;
    if (pending[b]) {
      cudaStreamWaitEvent(s, N->ev_buf[b], 0);
      pending[b] = false;
    }
    return dbuf[b];
  };
  auto advance = [&]() {
    ci = (ci + 1) % 3;
    dcur = dbuf[ci];
  };
  dother = next_out();
  HeadArgs hd{};
  hd.h = act_ptr(N, L);
  hd.gr = h.gr; hd.gc = h.gc; hd.vr = h.vr; hd.vc = h.vc; hd.Ch = h.C; hd.F = h.F;
  hd.w = N->params + N->lp[L].w_off;
  hd.b = N->params + N->lp[L].b_off;
  hd.C = N->classes;
  hd.hidden_act = N->lp[L - 1].L.act;
  hd.labels = d_labels;
  hd.O_H = N->O_H; hd.O_W = N->O_W;
  hd.n_levels = N->n_levels;
  for (int i = 0; i < N->n_levels; ++i) hd.pool_k[i] = N->pool_k[i];
  hd.nlab = nlab;
  for (int c = 0; c < 16; ++c) hd.cw[c] = (h_class_w && c < N->classes) ? h_class_w[c] : 1.f;
  hd.probs = nullptr;
  hd.dh = dcur;
  hd.loss_part = lossp;
  hd.part = bpart;
  hd.tiles_per_img = head_tiles_per_image((long long)h.F * h.gr * h.gc);
  hd.n_blocks = head_blocks((long long)hd.tiles_per_img * n);
  hd.err = (int*)(N->scratch + N->off_err);
  hd.n = n;
  hd.round_tf32 = tf32 ? 1 : 0;
  hd.zpre = N->z_ready ? scr(N, N->off_z) : nullptr;
  {
    const double pos = (double)n * h.F * h.vr * h.vc;
    uint8_t* labf = (uint8_t*)(N->scratch + N->off_labfrag);
    LAUNCH(N, s, "label_frag", L, 0.0, (double)n * h.F * h.gr * h.gc + (double)n * N->O_H * N->O_W,
           launch_label_frag(hd, labf, s));
    hd.lab_frag = labf;
    LAUNCH(N, s, "head_loss_delta", L, (hd.zpre ? 4.0 : 6.0) * pos * h.C * N->classes,
           pos * (8.0 * h.C + 1.0 + (hd.zpre ? 4.0 * N->classes : 0.0)), launch_head2(hd, s));
    const int E = N->classes * h.C + N->classes + h.C;
    if (loss_only) {  // forward-only loss evaluation (Armijo trial points): no gradients
      if (d_loss)
        LAUNCH(N, s, "loss_finalize", L, 0.0, 4.0 * (double)N->loss_parts * n,
               launch_loss_finalize(lossp, hd.tiles_per_img * head_loss_parts_per_tile(), nlab, n, d_loss,
                                  scr(N, N->off_lossred), (unsigned*)scr(N, N->off_lossred + sizeof(float) * kLossChunks * N->n_cap), s));
      return MPF_OK;
    }
    // [dW_L | db_L] are contiguous in the canonical order; db of layer L-1 follows
    LAUNCH(N, s, "head_reduce", L, 0.0, 4.0 * (double)hd.n_blocks * E,
           launch_partial_reduce(bpart, hd.n_blocks, E, N->grads + N->lp[L].w_off, N->grads + N->lp[L - 1].b_off,
                                 N->classes * h.C + N->classes, red_scratch(N, 0), s));
    if (d_loss)
      LAUNCH(N, s, "loss_finalize", L, 0.0, 4.0 * (double)N->loss_parts * n,
             launch_loss_finalize(lossp, hd.tiles_per_img * head_loss_parts_per_tile(), nlab, n, d_loss,
                                  scr(N, N->off_lossred), (unsigned*)scr(N, N->off_lossred + sizeof(float) * kLossChunks * N->n_cap), s));
  }
  // remaining layers in reverse.  Invariant: dcur holds the delta of a[l+1] at the
  // pre-activation (CONV/FC output) or the value (pooled output).
  long long hook_end = N->n_params;  // gradient entries [hook_end, n_params) already reported
  int bucket = 0;                    // index of the next gradient bucket (exchange flags)
  bool bias_done = true;  // layer L-1's bias came from the head
  bool premul = false;    // dcur already carries act' of the conv feeding the next pool
  float* wpack = scr(N, N->off_wpack);
  for (int l = L - 1; l >= 0; --l) {
    const LayerPlan& P = N->lp[l];
    const Act& in = N->a[l];
    const Act& o = N->a[l + 1];
    if (P.L.kind == MPF_POOL) {
      // Alg. 4: route deltas through mpIDXS, accumulate shared maxima; times act' of the
      // conv; the same pass sums the bias gradient of that conv (layer l-1)
      MpfBwdArgs m{};
      m.dout = dcur;
      m.pooled = tape_val(N, l);
      m.idx = tape_idx(N, l);
      m.gr = in.gr; m.gc = in.gc; m.vr = in.vr; m.vc = in.vc; m.C = in.C; m.k = P.L.k;
      m.m_r = o.vr; m.m_c = o.vc;
      m.n_frag_in = n * in.F;
      m.act = N->lp[l - 1].L.act;
      m.din = dother;
      m.round_tf32 = tf32 ? 1 : 0;
      m.bias_part = bpart;
      m.premul = premul ? 1 : 0;
      m.block_form = (N->cfg.flags & MPF_FLAG_MPF_BWD_BLOCK) ? 1 : 0;
      m.scatter_form = (N->cfg.flags & MPF_FLAG_MPF_BWD_SCATTER) ? 1 : 0;
      premul = false;
      const double ein = (double)n * in.F * in.vr * in.vc * in.C, eout = (double)n * o.F * o.vr * o.vc * o.C;
      LAUNCH(N, s, "mpf_bwd", l, 0.0, (m.premul ? 5.0 : 9.0) * eout + 4.0 * ein, launch_mpf_bwd(m, s));
      mpf_status st = bias_reduce(N, l - 1, bpart, mpf_bwd_partials(m), s);
      if (st != MPF_OK) return st;
      bias_done = true;
      advance();
      dother = next_out();
      continue;
    }
    if (!bias_done) {  // delta came from a dgrad (conv followed by conv)
      const long long Pp = (long long)n * o.F * o.gr * o.gc;
      LAUNCH(N, s, "bias_partial", l, 0.0, 4.0 * (double)Pp * P.cout,
             launch_channel_partial(dcur, Pp, P.cout, bpart, s));
      mpf_status st = bias_reduce(N, l, bpart, channel_partials(Pp), s);
      if (st != MPF_OK) return st;
    }
    bias_done = false;
    const float* x = (l == 0) ? N->images : act_ptr(N, l);
    if (sw != s) {  // the weight gradient of layer l on the side stream, after dcur is ready
      MPF_CUDA(cudaEventRecord(N->ev_ready, s));
      MPF_CUDA(cudaStreamWaitEvent(sw, N->ev_ready, 0));
    }
    mpf_status st = wgrad(N, l, x, dcur, n, sw);
    if (st != MPF_OK) return st;
    if (sw != s) {
      MPF_CUDA(cudaEventRecord(N->ev_buf[ci], sw));
      pending[ci] = true;
    }
    // every W / b of layers l .. L is final in the order of sw: one gradient bucket
    if (N->ex_on && N->ex_in_bwd)  // into every rank's exchange buffer, overlapping the rest
      MPF_CUDA(launch_exchange_push(N->grads, P.w_off, hook_end - P.w_off, N->ex_own, N->ex_layout, N->ex_rank,
                                    bucket, sw));
    if (N->grad_hook) N->grad_hook(N->grad_hook_user, l, P.w_off, hook_end - P.w_off, (void*)sw);
    hook_end = P.w_off;
    ++bucket;
    if (l == 0) break;
    // dgrad: delta of a[l] = full correlation of dcur with the rotated kernel.  When a[l]
    // is a pooled tensor, the epilogue already multiplies by act'(pooled value) of the conv
    // before that pool (= act'(y) at every element the pool selected), so the MPF backward
    // only routes and sums (premul).
    const bool in_is_conv = N->lp[l - 1].L.kind != MPF_POOL;
    const bool in_is_pool = !in_is_conv && l >= 2 && N->lp[l - 2].L.kind != MPF_POOL;
    const float* md = in_is_conv ? act_ptr(N, l) : (in_is_pool ? act_ptr(N, l) : nullptr);
    const int mdact = in_is_conv ? N->lp[l - 1].L.act : (in_is_pool ? N->lp[l - 2].L.act : 0);
    const double pos_out = (double)n * o.F * o.vr * o.vc, pos_in = (double)n * in.F * in.vr * in.vc;
    const double dflops = 2.0 * pos_out * P.cout * P.L.k * P.L.k * P.cin;
    const double dbytes = 4.0 * (pos_out * P.cout + pos_in * P.cin) + (md ? 4.0 * pos_in * P.cin : 0.0);
    if (use_tc(N, P, true)) {
      TcConvArgs t{};
      t.x = dcur; t.n_frag = n * in.F; t.gr = in.gr; t.gc = in.gc; t.cin = P.cout;
      t.w = wpack + P.dpack_off; t.bias = nullptr; t.k = P.L.k; t.cout = P.cin;
      t.out = dother; t.out_vr = in.vr; t.out_vc = in.vc; t.act = MPF_IDENTITY; t.shift = -(P.L.k - 1);
      t.round_out = (tf32 && !in_is_pool) ? 1 : 0;  // a pooled delta feeds the MPF backward, not an MMA
      t.zero_pad = 1;
      t.mul_dact = md;
      t.dact = mdact;
      t.flags = N->cfg.flags;
      LAUNCH(N, s, "dgrad_tc", l, dflops, dbytes, launch_conv_tc(t, s));
    } else {
      ConvArgs c{};
      c.in = dcur;
      c.in_F = in.F;
      c.image_mode = 0;
      c.in_gr = o.gr; c.in_gc = o.gc; c.in_vr = o.vr; c.in_vc = o.vc;
      c.off_y = c.off_x = -(P.L.k - 1);
      c.cin = P.cout;
      c.w = wpack + P.dpack_off;
      c.bias = nullptr;
      c.k = P.L.k;
      c.cout = P.cin;
      c.out = dother;
      c.out_gr = in.gr; c.out_gc = in.gc; c.out_vr = in.vr; c.out_vc = in.vc;
      c.act = MPF_IDENTITY;
      c.mul_dact = md;
      c.dact = mdact;
      c.zero_pad = 1;
      c.round_tf32 = (tf32 && !in_is_pool) ? 1 : 0;
      c.n_frag_total = n * in.F;
      LAUNCH(N, s, "dgrad_simt", l, dflops, dbytes, launch_conv_simt(c, s));
    }
    premul = in_is_pool;
    advance();
    dother = next_out();
  }
  if (sw != s) {  // the gradients are complete when the side stream is
    MPF_CUDA(cudaEventRecord(N->ev_join, sw));
    MPF_CUDA(cudaStreamWaitEvent(s, N->ev_join, 0));
  }
  return MPF_OK;
}

mpf_status mpf_backward_image(mpf_net* N, const uint8_t* d_labels, const float* h_class_w, float* d_loss,
                              void* stream) {
  if (!N || !d_labels) return fail(MPF_ERR_ARG, "NULL argument");
  if (!N->bound) return fail(MPF_ERR_STATE, "net is not bound");
  if (!N->have_fwd) return fail(MPF_ERR_STATE, "mpf_backward_image before mpf_forward_image");
  NvtxRange nv("mpf_backward_image", N->n_fwd);
  return backward_impl(N, d_labels, h_class_w, d_loss, (cudaStream_t)stream);
}

mpf_status mpf_train_step(mpf_net* N, const float* d_images, int32_t n, const uint8_t* d_labels,
                          const float* h_class_w, float* d_loss, void* stream) {
  if (!N || !d_images || !d_labels) return fail(MPF_ERR_ARG, "NULL argument");
  if (!N->bound) return fail(MPF_ERR_STATE, "net is not bound (mpf_net_bind)");
  if (n < 1 || n > N->n_cap) return fail(MPF_ERR_DATA, "n must be in [1, bound n_images]");
  cudaStream_t s = (cudaStream_t)stream;
  NvtxRange nv("mpf_train_step", n);
  mpf_status st = forward_impl(N, d_images, n, nullptr, s);
  if (st != MPF_OK) return st;
  return backward_impl(N, d_labels, h_class_w, d_loss, s);
}

// Armijo-safeguarded gradient step ("stochastic gradient descent safe-guarded
// by the Armijo rule"): g = grad_scale * (sum of the images' gradients),
// d = -g, alpha = alpha0, alpha0 beta, ... until L(theta + alpha d) <= L(theta) - c alpha ||g||^2
// with L = grad_scale * (sum of the images' losses); trial points are forward-only loss
// evaluations (forward + the head's loss).  Accepted: theta moves; exhausted: theta unchanged.
// The gradient buffer is zeroed either way.  h_out[5] = {L0, L_final, alpha (0 if rejected),
// accepted, loss evaluations}.  Synchronises the stream once per trial (the line search is a
// host decision).
mpf_status mpf_armijo_step(mpf_net* N, const float* d_images, int32_t n, const uint8_t* d_labels,
                           const float* h_class_w, float alpha0, float beta, float c, int32_t max_backtracks,
                           float grad_scale, float* h_out, void* stream) {
  if (!N || !d_images || !d_labels || !h_out) return fail(MPF_ERR_ARG, "NULL argument");
  if (!N->bound) return fail(MPF_ERR_STATE, "net is not bound");
  if (n < 1 || n > N->n_cap) return fail(MPF_ERR_DATA, "n must be in [1, bound n_images]");
  if (!(alpha0 > 0.f) || !(beta > 0.f && beta < 1.f) || !(c > 0.f && c < 1.f) || max_backtracks < 0)
    return fail(MPF_ERR_ARG, "Armijo parameters: alpha0 > 0, 0 < beta < 1, 0 < c < 1, max_backtracks >= 0");
  cudaStream_t s = (cudaStream_t)stream;
  float* d_loss = scr(N, N->off_stage_loss);
  float h_loss[256];
  if (n > 256) return fail(MPF_ERR_ARG, "at most 256 images per Armijo step");
  auto total_loss = [&](double* L) -> mpf_status {
    MPF_CUDA(cudaMemcpyAsync(h_loss, d_loss, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
    MPF_CUDA(cudaStreamSynchronize(s));
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += h_loss[i];
    *L = t * grad_scale;
    return MPF_OK;
  };
  // 1. loss and gradient at theta (the buffer is zeroed first: leftovers, e.g. the last
  // trial's gradient of mpf_lbfgs_step, must not enter g)
  MPF_CUDA(cudaMemsetAsync(N->grads, 0, sizeof(float) * N->n_params, s));
  mpf_status st = mpf_train_step(N, d_images, n, d_labels, h_class_w, d_loss, stream);
  if (st != MPF_OK) return st;
  double L0 = 0.0, g2 = 0.0;
  double* d_parts = (double*)(N->scratch + N->off_armijo);
  MPF_CUDA(launch_sqnorm(N->grads, N->n_params, d_parts, kArmijoParts, d_parts + kArmijoParts, s));
  MPF_CUDA(cudaMemcpyAsync(&g2, d_parts + kArmijoParts, sizeof(double), cudaMemcpyDeviceToHost, s));
  st = total_loss(&L0);
  if (st != MPF_OK) return st;
  g2 *= (double)grad_scale * grad_scale;
  if (!std::isfinite(L0) || !std::isfinite(g2)) {
    MPF_CUDA(cudaMemsetAsync(N->grads, 0, sizeof(float) * N->n_params, s));
    return fail(MPF_ERR_DATA, "Armijo: non-finite loss or gradient");
  }
  // 2. backtracking along d = -g from the saved base point
  float* theta0 = scr(N, N->off_theta0);
  MPF_CUDA(cudaMemcpyAsync(theta0, N->params, sizeof(float) * N->n_params, cudaMemcpyDeviceToDevice, s));
  double alpha = alpha0, L = L0;
  int evals = 0;
  bool accepted = false;
  for (int it = 0; it <= max_backtracks; ++it, alpha *= beta) {
    MPF_CUDA(launch_armijo_axpy(N->params, theta0, N->grads, N->n_params, (float)(alpha * grad_scale), s));
    st = forward_impl(N, d_images, n, nullptr, s);
    if (st != MPF_OK) return st;
    st = backward_impl(N, d_labels, h_class_w, d_loss, s, true);
    if (st != MPF_OK) return st;
    st = total_loss(&L);
    if (st != MPF_OK) return st;
    ++evals;
    if (std::isfinite(L) && L <= L0 - (double)c * alpha * g2) {
      accepted = true;
      break;
    }
  }
  if (!accepted) {
    MPF_CUDA(cudaMemcpyAsync(N->params, theta0, sizeof(float) * N->n_params, cudaMemcpyDeviceToDevice, s));
    L = L0;
  }
  MPF_CUDA(cudaMemsetAsync(N->grads, 0, sizeof(float) * N->n_params, s));
  N->have_fwd = false;  // the tape holds a trial point
  h_out[0] = (float)L0;
  h_out[1] = (float)L;
  h_out[2] = accepted ? (float)alpha : 0.f;
  h_out[3] = accepted ? 1.f : 0.f;
  h_out[4] = (float)evals;
  return MPF_OK;
}

// ============================================================================ L-BFGS
// Full-batch L-BFGS (reading R21).  Device state lives in
// one allocation; the pair bookkeeping (which slots hold which pair, s^T y, y^T y) is on
// the host, which needs s^T y anyway to decide whether a pair is kept.
}  // extern "C"

constexpr int kLbParts = 592;  // blocks of every L-BFGS pass (148 SMs x 4)

struct mpf_lbfgs {
  mpf_net* N = nullptr;
  int m = 0;                    // memory (pairs kept)
  long long n = 0;              // parameters
  char* mem = nullptr;          // caller-owned device state (mpf_lbfgs_state_bytes)
  float* S = nullptr;           // (m+1) slots of s, then of y
  float* Y = nullptr;
  float* theta0 = nullptr;
  float* g = nullptr;           // grad_scale * gradient at theta0 / the current point
  double* v = nullptr;          // H g
  double* parts = nullptr;      // 2 x kLbParts partial sums (ping, pong)
  double* a = nullptr;          // alpha_i of the first loop, per slot
  std::vector<int> order;       // stored pairs' slots, oldest first
  std::vector<double> sy, yy;   // per slot
  bool have_g = false, have_dir = false;
  bool have_L = false;          // L is the loss at the point of g (set only by mpf_lbfgs_step)
  double L = 0.0;               // mpf_lbfgs_step: loss at the current point (valid with have_L)
  std::vector<double> hpart;
};

namespace {
double host_sum(const std::vector<double>& p, int off, int nb) {
  double t = 0.0;
  for (int i = 0; i < nb; ++i) t += p[off + i];
  return t;
}
}  // namespace

extern "C" {

static size_t lbfgs_bytes(long long n, int memory) {
  const size_t vec = align256(sizeof(float) * (size_t)n);
  const size_t slots = (size_t)memory + 1;
  return 2 * slots * vec + 2 * vec + align256(sizeof(double) * (size_t)n) + align256(sizeof(double) * 2 * kLbParts) +
         align256(sizeof(double) * slots);
}

mpf_status mpf_lbfgs_state_bytes(const mpf_net* N, int32_t memory, uint64_t* bytes) {
  if (!N || !bytes) return fail(MPF_ERR_ARG, "NULL argument");
  if (memory < 1 || memory > 64) return fail(MPF_ERR_ARG, "L-BFGS memory must be in [1, 64]");
  *bytes = lbfgs_bytes(N->n_params, memory);
  return MPF_OK;
}

mpf_status mpf_lbfgs_create(mpf_net* N, int32_t memory, void* d_state, uint64_t state_bytes, mpf_lbfgs** out) {
  if (!N || !out || !d_state) return fail(MPF_ERR_ARG, "NULL argument");
  if (memory < 1 || memory > 64) return fail(MPF_ERR_ARG, "L-BFGS memory must be in [1, 64]");
  if (!N->bound) return fail(MPF_ERR_STATE, "net is not bound");
  if (((uintptr_t)d_state & 255) != 0) return fail(MPF_ERR_ARG, "L-BFGS state must be 256-byte aligned");
  if (state_bytes < lbfgs_bytes(N->n_params, memory)) return fail(MPF_ERR_ARG, "L-BFGS state buffer too small");
  mpf_lbfgs* lb = new mpf_lbfgs();
  lb->N = N;
  lb->m = memory;
  lb->n = N->n_params;
  const size_t vec = align256(sizeof(float) * (size_t)lb->n);
  const size_t slots = (size_t)memory + 1;
  lb->mem = (char*)d_state;
  char* p = lb->mem;
  lb->S = (float*)p; p += slots * vec;
  lb->Y = (float*)p; p += slots * vec;
  lb->theta0 = (float*)p; p += vec;
  lb->g = (float*)p; p += vec;
  lb->v = (double*)p; p += align256(sizeof(double) * (size_t)lb->n);
  lb->parts = (double*)p; p += align256(sizeof(double) * 2 * kLbParts);
  lb->a = (double*)p;
  lb->sy.assign(slots, 0.0);
  lb->yy.assign(slots, 0.0);
  lb->hpart.assign(2 * kLbParts, 0.0);
  *out = lb;
  return MPF_OK;
}

void mpf_lbfgs_destroy(mpf_lbfgs* lb) { delete lb; }  // the state buffer belongs to the caller

mpf_status mpf_lbfgs_reset(mpf_lbfgs* lb) {
  if (!lb) return fail(MPF_ERR_ARG, "NULL L-BFGS state");
  lb->order.clear();
  lb->have_g = lb->have_dir = lb->have_L = false;
  return MPF_OK;
}

mpf_status mpf_lbfgs_set_gradient(mpf_lbfgs* lb, float grad_scale, void* stream) {
  if (!lb) return fail(MPF_ERR_ARG, "NULL L-BFGS state");
  MPF_CUDA(launch_lbfgs_gset(lb->g, lb->N->grads, lb->n, grad_scale, (cudaStream_t)stream));
  lb->have_g = true;
  lb->have_dir = false;
  lb->have_L = false;  // a caller-supplied gradient: its loss is not known here
  return MPF_OK;
}

mpf_status mpf_lbfgs_direction(mpf_lbfgs* lb, double* h_gtd, int32_t* h_fallback, void* stream) {
  if (!lb || !h_gtd) return fail(MPF_ERR_ARG, "NULL argument");
  if (!lb->have_g) return fail(MPF_ERR_STATE, "L-BFGS direction without a gradient (mpf_lbfgs_set_gradient)");
  cudaStream_t s = (cudaStream_t)stream;
  const int k = (int)lb->order.size();
  const long long n = lb->n;
  double* P[2] = {lb->parts, lb->parts + kLbParts};
  int cur = 0;
  auto slotS = [&](int j) { return lb->S + (size_t)lb->order[j] * (align256(sizeof(float) * n) / sizeof(float)); };
  auto slotY = [&](int j) { return lb->Y + (size_t)lb->order[j] * (align256(sizeof(float) * n) / sizeof(float)); };
  // two-loop: q = g; newest -> oldest: a_i = rho_i s_i.q, q -= a_i y_i; r = gamma q;
  // oldest -> newest: b = rho_i y_i.r, r += (a_i - b) s_i.  Passes ping-pong the partials.
  MPF_CUDA(launch_lbfgs_pass(lb->v, lb->g, k ? slotS(k - 1) : lb->g, n, nullptr, 0, 0.0, nullptr, 1.0, P[cur],
                             kLbParts, s));
  if (k) {
    const int newest = lb->order[k - 1];
    const double gamma = lb->sy[newest] / lb->yy[newest];
    for (int j = k - 1; j >= 0; --j) {
      const int sl = lb->order[j];
      const float* z = j > 0 ? slotS(j - 1) : slotY(0);
      MPF_CUDA(launch_lbfgs_pass(lb->v, slotY(j), z, n, P[cur], 1, 1.0 / lb->sy[sl], lb->a + sl,
                                 j == 0 ? gamma : 1.0, P[cur ^ 1], kLbParts, s));
      cur ^= 1;
    }
    for (int j = 0; j < k; ++j) {
      const int sl = lb->order[j];
      const float* z = j < k - 1 ? slotY(j + 1) : lb->g;
      MPF_CUDA(launch_lbfgs_pass(lb->v, slotS(j), z, n, P[cur], 2, 1.0 / lb->sy[sl], lb->a + sl, 1.0,
                                 P[cur ^ 1], kLbParts, s));
      cur ^= 1;
    }
  }
  MPF_CUDA(cudaMemcpyAsync(lb->hpart.data(), P[cur], sizeof(double) * kLbParts, cudaMemcpyDeviceToHost, s));
  MPF_CUDA(cudaMemcpyAsync(lb->theta0, lb->N->params, sizeof(float) * n, cudaMemcpyDeviceToDevice, s));
  MPF_CUDA(cudaStreamSynchronize(s));
  double gtd = -host_sum(lb->hpart, 0, kLbParts);  // d = -v
  int fb = 0;
  if (!(gtd < 0.0)) {  // not a descent direction (or not finite): steepest descent
    fb = 1;
    MPF_CUDA(launch_lbfgs_pass(lb->v, lb->g, lb->g, n, nullptr, 0, 0.0, nullptr, 1.0, P[0], kLbParts, s));
    MPF_CUDA(cudaMemcpyAsync(lb->hpart.data(), P[0], sizeof(double) * kLbParts, cudaMemcpyDeviceToHost, s));
    MPF_CUDA(cudaStreamSynchronize(s));
    gtd = -host_sum(lb->hpart, 0, kLbParts);
  }
  *h_gtd = gtd;
  if (h_fallback) *h_fallback = fb;
  lb->have_dir = true;
  return MPF_OK;
}

mpf_status mpf_lbfgs_trial(mpf_lbfgs* lb, double alpha, void* stream) {
  if (!lb) return fail(MPF_ERR_ARG, "NULL L-BFGS state");
  if (!lb->have_dir) return fail(MPF_ERR_STATE, "L-BFGS trial without a direction");
  MPF_CUDA(launch_lbfgs_trial(lb->N->params, lb->theta0, lb->v, lb->n, alpha, (cudaStream_t)stream));
  return MPF_OK;
}

mpf_status mpf_lbfgs_accept(mpf_lbfgs* lb, float grad_scale, int32_t* h_stored, void* stream) {
  if (!lb) return fail(MPF_ERR_ARG, "NULL L-BFGS state");
  if (!lb->have_dir) return fail(MPF_ERR_STATE, "L-BFGS accept without a direction");
  cudaStream_t s = (cudaStream_t)stream;
  const long long n = lb->n;
  const size_t stride = align256(sizeof(float) * n) / sizeof(float);
  int slot = 0;  // a slot no stored pair uses (there are memory + 1)
  for (; slot <= lb->m; ++slot) {
    bool used = false;
    for (int o : lb->order) used |= (o == slot);
    if (!used) break;
  }
  double* part = lb->parts;  // s.y partials, then y.y partials
  MPF_CUDA(launch_lbfgs_pair(lb->S + slot * stride, lb->Y + slot * stride, lb->g, lb->N->params, lb->theta0,
                             lb->N->grads, n, grad_scale, part, kLbParts, s));
  MPF_CUDA(cudaMemcpyAsync(lb->hpart.data(), part, sizeof(double) * 2 * kLbParts, cudaMemcpyDeviceToHost, s));
  MPF_CUDA(cudaStreamSynchronize(s));
  const double sy = host_sum(lb->hpart, 0, kLbParts), yy = host_sum(lb->hpart, kLbParts, kLbParts);
  const bool keep = sy > 1e-10 && std::isfinite(sy) && std::isfinite(yy);
  if (keep) {
    if ((int)lb->order.size() == lb->m) lb->order.erase(lb->order.begin());
    lb->order.push_back(slot);
    lb->sy[slot] = sy;
    lb->yy[slot] = yy;
  }
  if (h_stored) *h_stored = keep ? 1 : 0;
  lb->have_g = true;
  lb->have_dir = false;
  return MPF_OK;
}

mpf_status mpf_lbfgs_reject(mpf_lbfgs* lb, void* stream) {
  if (!lb) return fail(MPF_ERR_ARG, "NULL L-BFGS state");
  if (!lb->have_dir) return fail(MPF_ERR_STATE, "L-BFGS reject without a direction");
  MPF_CUDA(cudaMemcpyAsync(lb->N->params, lb->theta0, sizeof(float) * lb->n, cudaMemcpyDeviceToDevice,
                           (cudaStream_t)stream));
  lb->order.clear();
  lb->have_dir = false;  // g still holds the gradient at theta0
  return MPF_OK;
}

mpf_status mpf_line_search_first(double alpha0, int32_t n_pairs, double* alpha) {
  if (!alpha) return fail(MPF_ERR_ARG, "NULL argument");
  *alpha = n_pairs == 0 ? alpha0 : 1.0;
  return MPF_OK;
}

mpf_status mpf_line_search_decide(double L0, double gtd, double c, double beta, double alpha, double L_trial,
                                  int32_t trials_done, int32_t max_backtracks, int32_t* decision,
                                  double* alpha_next) {
  if (!decision || !alpha_next) return fail(MPF_ERR_ARG, "NULL argument");
  if (!(beta > 0.0 && beta < 1.0) || !(c > 0.0 && c < 1.0) || max_backtracks < 0 || trials_done < 1)
    return fail(MPF_ERR_ARG, "line search: 0 < beta < 1, 0 < c < 1, max_backtracks >= 0, trials_done >= 1");
  *alpha_next = alpha;
  if (std::isfinite(L_trial) && L_trial <= L0 + c * alpha * gtd) *decision = 1;  // Armijo: sufficient decrease
  else if (trials_done > max_backtracks) *decision = -1;
  else {
    *decision = 0;
    *alpha_next = beta * alpha;
  }
  return MPF_OK;
}

mpf_status mpf_lbfgs_step(mpf_lbfgs* lb, const float* d_images, int32_t n, const uint8_t* d_labels,
                          const float* h_class_w, float alpha0, float beta, float c, int32_t max_backtracks,
                          float grad_scale, float* h_out, void* stream) {
  if (!lb || !d_images || !d_labels || !h_out) return fail(MPF_ERR_ARG, "NULL argument");
  mpf_net* N = lb->N;
  if (n < 1 || n > N->n_cap) return fail(MPF_ERR_DATA, "n must be in [1, bound n_images]");
  if (n > 256) return fail(MPF_ERR_ARG, "at most 256 images per L-BFGS evaluation");
  if (!(alpha0 > 0.f) || !(beta > 0.f && beta < 1.f) || !(c > 0.f && c < 1.f) || max_backtracks < 0)
    return fail(MPF_ERR_ARG, "line search parameters: alpha0 > 0, 0 < beta < 1, 0 < c < 1, max_backtracks >= 0");
  cudaStream_t s = (cudaStream_t)stream;
  float* d_loss = scr(N, N->off_stage_loss);
  float h_loss[256];
  // loss and gradient of the full batch at the current parameters
  auto evaluate = [&](double* L) -> mpf_status {
    MPF_CUDA(cudaMemsetAsync(N->grads, 0, sizeof(float) * N->n_params, s));
    mpf_status st = mpf_train_step(N, d_images, n, d_labels, h_class_w, d_loss, stream);
    if (st != MPF_OK) return st;
    MPF_CUDA(cudaMemcpyAsync(h_loss, d_loss, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
    MPF_CUDA(cudaStreamSynchronize(s));
    double t = 0.0;
    for (int i = 0; i < n; ++i) t += h_loss[i];
    *L = t * grad_scale;
    return MPF_OK;
  };
  mpf_status st;
  if (!lb->have_g || !lb->have_L) {  // first call, after a reset or after a caller-supplied gradient
    double L0 = 0.0;
    st = evaluate(&L0);
    if (st != MPF_OK) return st;
    st = mpf_lbfgs_set_gradient(lb, grad_scale, stream);
    if (st != MPF_OK) return st;
    lb->L = L0;
    lb->have_L = true;
  }
  const double L0 = lb->L;
  double gtd = 0.0;
  int32_t fb = 0;
  st = mpf_lbfgs_direction(lb, &gtd, &fb, stream);
  if (st != MPF_OK) return st;
  if (!std::isfinite(L0) || !std::isfinite(gtd)) {
    lb->have_g = lb->have_dir = lb->have_L = false;
    return fail(MPF_ERR_DATA, "L-BFGS: non-finite loss or direction");
  }
  double alpha = 0.0, L = L0;
  mpf_line_search_first(alpha0, (int32_t)lb->order.size(), &alpha);
  int evals = 0;
  bool accepted = false;
  for (;;) {
    st = mpf_lbfgs_trial(lb, alpha, stream);
    if (st != MPF_OK) return st;
    st = evaluate(&L);
    if (st != MPF_OK) return st;
    ++evals;
    int32_t decision = 0;
    double next = 0.0;
    st = mpf_line_search_decide(L0, gtd, c, beta, alpha, L, evals, max_backtracks, &decision, &next);
    if (st != MPF_OK) return st;
    if (decision != 0) {
      accepted = decision == 1;
      break;
    }
    alpha = next;
  }
  if (accepted) {
    st = mpf_lbfgs_accept(lb, grad_scale, nullptr, stream);
    if (st != MPF_OK) return st;
    lb->L = L;
  } else {
    st = mpf_lbfgs_reject(lb, stream);
    if (st != MPF_OK) return st;
    L = L0;
  }
  N->have_fwd = false;
  h_out[0] = (float)L0;
  h_out[1] = (float)L;
  h_out[2] = accepted ? (float)alpha : 0.f;
  h_out[3] = accepted ? 1.f : 0.f;
  h_out[4] = (float)evals;
  h_out[5] = (float)fb;
  h_out[6] = (float)lb->order.size();
  return MPF_OK;
}

// gradient buckets one backward reports (conv / FC layers but the softmax FC, which goes with
// the last hidden layer's bucket)
static int n_grad_buckets(const mpf_net* N) {
  int nb = 0;
  for (int l = 0; l < N->n_layers; ++l) nb += N->lp[l].L.kind != MPF_POOL;
  return nb > 1 ? nb - 1 : 1;
}

mpf_status mpf_exchange_bytes(const mpf_net* N, int32_t world, size_t* bytes) {
  if (!N || !bytes) return fail(MPF_ERR_ARG, "NULL argument");
  if (world < 1 || world > ExLayout::kMaxWorld) return fail(MPF_ERR_ARG, "world out of range [1, 64]");
  *bytes = exchange_layout(world, N->n_layers, N->n_params).bytes;
  return MPF_OK;
}

mpf_status mpf_exchange_attach(mpf_net* N, int32_t rank, int32_t world, void* const* d_bufs, int32_t push_in_backward) {
  if (!N || !d_bufs) return fail(MPF_ERR_ARG, "NULL argument");
  if (!N->bound) return fail(MPF_ERR_STATE, "net is not bound (mpf_net_bind)");
  if (world < 1 || world > ExLayout::kMaxWorld) return fail(MPF_ERR_ARG, "world out of range [1, 64]");
  if (rank < 0 || rank >= world) return fail(MPF_ERR_ARG, "rank out of range [0, world)");
  uint64_t peers[ExLayout::kMaxWorld];
  for (int r = 0; r < world; ++r) {
    if (!d_bufs[r]) return fail(MPF_ERR_ARG, "NULL exchange buffer of rank " + std::to_string(r));
    if ((uintptr_t)d_bufs[r] % 256) return fail(MPF_ERR_ARG, "exchange buffers must be 256-byte aligned");
    peers[r] = (uint64_t)(uintptr_t)d_bufs[r];
  }
  N->ex_layout = exchange_layout(world, N->n_layers, N->n_params);
  N->ex_own = (char*)d_bufs[rank];
  N->ex_rank = rank;
  N->ex_in_bwd = push_in_backward != 0;
  MPF_CUDA(cudaMemcpy(N->ex_own + ExLayout::kPeers, peers, sizeof(uint64_t) * world, cudaMemcpyHostToDevice));
  N->ex_on = true;
  return MPF_OK;
}

mpf_status mpf_exchange_detach(mpf_net* N) {
  if (!N) return fail(MPF_ERR_ARG, "NULL net");
  N->ex_on = false;
  N->ex_own = nullptr;
  return MPF_OK;
}

mpf_status mpf_exchange_push(mpf_net* N, void* stream) {
  if (!N) return fail(MPF_ERR_ARG, "NULL net");
  if (!N->ex_on) return fail(MPF_ERR_STATE, "no exchange attached (mpf_exchange_attach)");
  if (N->ex_in_bwd) return fail(MPF_ERR_STATE, "the backward pushes (attached with push_in_backward = 1)");
  cudaStream_t s = (cudaStream_t)stream;
  LAUNCH(N, s, "exchange_push", -1, 0.0, 4.0 * (1 + N->ex_layout.world) * N->n_params,
         launch_exchange_push(N->grads, 0, N->n_params, N->ex_own, N->ex_layout, N->ex_rank, 0, s));
  return MPF_OK;
}

mpf_status mpf_exchange_sgd_step(mpf_net* N, float lr, float scale, void* stream) {
  if (!N) return fail(MPF_ERR_ARG, "NULL net");
  if (!N->bound) return fail(MPF_ERR_STATE, "net is not bound");
  if (!N->ex_on) return fail(MPF_ERR_STATE, "no exchange attached (mpf_exchange_attach)");
  cudaStream_t s = (cudaStream_t)stream;
  const int nb = N->ex_in_bwd ? n_grad_buckets(N) : 1;
  LAUNCH(N, s, "exchange_sgd", -1, (1.0 + N->ex_layout.world) * N->n_params,
         4.0 * (N->ex_layout.world + 3) * N->n_params,
         launch_exchange_sgd(N->params, N->grads, lr, scale, N->ex_own, N->ex_layout, nb, s));
  return MPF_OK;
}

mpf_status mpf_sgd_step(mpf_net* N, float lr, float scale, void* stream) {
  if (!N) return fail(MPF_ERR_ARG, "NULL net");
  if (!N->bound) return fail(MPF_ERR_STATE, "net is not bound");
  if (N->ex_on) return mpf_exchange_sgd_step(N, lr, scale, stream);
  cudaStream_t s = (cudaStream_t)stream;
  LAUNCH(N, s, "sgd", -1, 2.0 * N->n_params, 16.0 * N->n_params,
         launch_sgd(N->params, N->grads, N->n_params, lr, scale, s));
  return MPF_OK;
}

mpf_status mpf_train_step_host(mpf_net* N, const float* h_images, const uint8_t* h_labels, int32_t n,
                               const float* h_class_w, float* h_loss, int32_t apply_sgd, float lr, float scale,
                               void* stream) {
  if (!N || !h_images || !h_labels) return fail(MPF_ERR_ARG, "NULL argument");
  if (!N->bound) return fail(MPF_ERR_STATE, "net is not bound");
  if (n < 1 || n > N->n_cap) return fail(MPF_ERR_DATA, "n must be in [1, bound n_images]");
  cudaStream_t s = (cudaStream_t)stream;
  // Double-buffered inputs: this step's H2D copies run on a copy stream into staging slot
  // b, after the step that last read slot b (two calls ago) has finished with it; the
  // compute stream waits only for its own slot.  Consecutive calls therefore overlap the
  // next step's upload with this step's kernels (both inside a caller's timing of the
  // calls), and the results are those of the serial order.
  if (!N->copy_stream) {
    MPF_CUDA(cudaStreamCreateWithFlags(&N->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      MPF_CUDA(cudaEventCreateWithFlags(&N->ev_copied[i], cudaEventDisableTiming));
      MPF_CUDA(cudaEventCreateWithFlags(&N->ev_free[i], cudaEventDisableTiming));
      MPF_CUDA(cudaEventRecord(N->ev_free[i], s));
    }
  }
  const int b = N->stage_slot;
  N->stage_slot ^= 1;
  float* d_img = scr(N, N->off_stage_img + b * N->stage_bytes);
  uint8_t* d_lab = (uint8_t*)(N->scratch + N->off_stage_lab + b * N->stage_bytes);
  float* d_loss = scr(N, N->off_stage_loss);
  const size_t ib = sizeof(float) * (size_t)n * N->cfg.in_channels * N->cfg.image_rows * N->cfg.image_cols;
  const size_t lb = (size_t)n * N->O_H * N->O_W;
  MPF_CUDA(cudaStreamWaitEvent(N->copy_stream, N->ev_free[b], 0));
  MPF_CUDA(cudaMemcpyAsync(d_img, h_images, ib, cudaMemcpyHostToDevice, N->copy_stream));
  MPF_CUDA(cudaMemcpyAsync(d_lab, h_labels, lb, cudaMemcpyHostToDevice, N->copy_stream));
  MPF_CUDA(cudaEventRecord(N->ev_copied[b], N->copy_stream));
  MPF_CUDA(cudaStreamWaitEvent(s, N->ev_copied[b], 0));
  mpf_status st = mpf_train_step(N, d_img, n, d_lab, h_class_w, d_loss, stream);
  if (st != MPF_OK) return st;
  MPF_CUDA(cudaEventRecord(N->ev_free[b], s));  // slot b's images / labels are consumed
  if (apply_sgd) {
    st = mpf_sgd_step(N, lr, scale, stream);
    if (st != MPF_OK) return st;
  }
  if (h_loss) MPF_CUDA(cudaMemcpyAsync(h_loss, d_loss, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
  return MPF_OK;
}

mpf_status mpf_mirror_pad(const float* d_in, int32_t planes, int32_t rows, int32_t cols, int32_t pad_top,
                          int32_t pad_left, int32_t out_rows, int32_t out_cols, float* d_out, void* stream) {
  if (!d_in || !d_out) return fail(MPF_ERR_ARG, "NULL argument");
  if (planes < 1 || rows < 1 || cols < 1 || pad_top < 0 || pad_left < 0) return fail(MPF_ERR_ARG, "bad sizes");
  const int pb = out_rows - rows - pad_top, pr = out_cols - cols - pad_left;
  if (pb < 0 || pr < 0) return fail(MPF_ERR_ARG, "output smaller than input + leading pads");
  if (pad_top >= rows || pad_left >= cols || pb >= rows || pr >= cols)
    return fail(MPF_ERR_ARG, "a pad must be smaller than the image (single reflection)");
  MPF_CUDA(launch_mirror_pad(d_in, d_out, planes, rows, cols, pad_top, pad_left, out_rows, out_cols,
                             (cudaStream_t)stream));
  return MPF_OK;
}

mpf_status mpf_class_weights_auto(const mpf_net* N, const uint8_t* d_labels, int32_t n, float* h_class_w,
                                  uint64_t* h_counts, void* stream) {
  if (!N || !d_labels || !h_class_w) return fail(MPF_ERR_ARG, "NULL argument");
  if (!N->bound) return fail(MPF_ERR_STATE, "net is not bound");
  if (n < 1) return fail(MPF_ERR_ARG, "n must be >= 1");
  cudaStream_t s = (cudaStream_t)stream;
  const int C = N->classes;
  // the counts go to the loss-partials region of the scratch (free between steps)
  unsigned long long* d_counts = (unsigned long long*)(N->scratch + N->off_lossp);
  if (sizeof(unsigned long long) * C > sizeof(float) * (size_t)N->loss_parts * N->n_cap)
    return fail(MPF_ERR_INTERNAL, "scratch too small for the class histogram");
  MPF_CUDA(launch_class_hist(d_labels, (long long)n * N->O_H * N->O_W, C, d_counts, s));
  unsigned long long h[256];
  MPF_CUDA(cudaMemcpyAsync(h, d_counts, sizeof(unsigned long long) * C, cudaMemcpyDeviceToHost, s));
  MPF_CUDA(cudaStreamSynchronize(s));
  unsigned long long tot = 0;
  for (int c = 0; c < C; ++c) tot += h[c];
  for (int c = 0; c < C; ++c) {
    if (h_counts) h_counts[c] = h[c];
    if (h[c] == 0)
      return fail(MPF_ERR_DATA, "auto class weights: class " + std::to_string(c) + " has no labelled pixel");
  }
  for (int c = 0; c < C; ++c) h_class_w[c] = (float)((double)tot / ((double)C * (double)h[c]));
  return MPF_OK;
}

mpf_status mpf_fragments_to_pixels(const mpf_net* N, const float* d_frag, float* d_pix, int32_t n, int32_t C,
                                   void* stream) {
  if (!N || !d_frag || !d_pix) return fail(MPF_ERR_ARG, "NULL argument");
  if (n < 1 || C < 1) return fail(MPF_ERR_ARG, "n and channels must be >= 1");
  const Act& o = N->a[N->n_layers];
  cudaStream_t s = (cudaStream_t)stream;
  Net* Nm = const_cast<mpf_net*>(N);
  LAUNCH(Nm, s, "frag2pix", -1, 0.0, 8.0 * n * C * N->O_H * N->O_W,
         launch_frag2pix(d_frag, d_pix, n, C, o.F, o.vr, o.vc, N->O_H, N->O_W, N->n_levels, N->pool_k, s));
  return MPF_OK;
}

mpf_status mpf_debug_tape(const mpf_net* N, int32_t layer, int32_t what, void* dst, void* stream) {
  if (!N || !dst) return fail(MPF_ERR_ARG, "NULL argument");
  if (!N->have_fwd) return fail(MPF_ERR_STATE, "no forward yet");
  if (layer < 0 || layer >= N->n_layers) return fail(MPF_ERR_ARG, "layer out of range");
  const LayerPlan& P = N->lp[layer];
  const Act& o = N->a[layer + 1];
  cudaStream_t s = (cudaStream_t)stream;
  const long long nf = (long long)N->n_fwd * o.F;
  if (what == MPF_TAPE_ARGMAX) {
    if (P.L.kind != MPF_POOL) return fail(MPF_ERR_ARG, "argmax exists only for POOL layers");
    MPF_CUDA(cudaMemcpyAsync(dst, tape_idx(N, layer), (size_t)nf * o.vr * o.vc * o.C, cudaMemcpyDeviceToDevice, s));
    return MPF_OK;
  }
  if (what != MPF_TAPE_VALUE) return fail(MPF_ERR_ARG, "unknown tape item");
  if (P.out_where != Where::Tape) return fail(MPF_ERR_ARG, "this layer's output is not kept on the tape");
  MPF_CUDA(launch_compact_copy(tape_val(N, layer), o.gr, o.gc, o.vr, o.vc, o.C, nf, (float*)dst, s));
  return MPF_OK;
}

mpf_status mpf_net_set_grad_hook(mpf_net* N, mpf_grad_ready_fn fn, void* user) {
  if (!N) return fail(MPF_ERR_ARG, "NULL net");
  N->grad_hook = fn;
  N->grad_hook_user = user;
  return MPF_OK;
}

mpf_status mpf_net_set_flags(mpf_net* N, uint32_t flags) {
  if (!N) return fail(MPF_ERR_ARG, "NULL net");
  const uint32_t known = MPF_FLAG_SERIAL | MPF_FLAG_TC_SINGLE | MPF_FLAG_TC_PAIR | MPF_FLAG_NTAP_ON | MPF_FLAG_NTAP_OFF |
                         MPF_FLAG_NTAP_NO_MC | MPF_FLAG_WGRAD_M128 | MPF_FLAG_ROLE_TIMERS | MPF_FLAG_FUSE_FIRST_POOL |
                         MPF_FLAG_HEAD_LOGITS_OFF | MPF_FLAG_HEAD_LOGITS_ON | MPF_FLAG_MPF_BWD_BLOCK |
                         MPF_FLAG_MPF_BWD_SCATTER;
  if (flags & ~known) return fail(MPF_ERR_ARG, "unknown MPF_FLAG_* bits");
  if ((flags & MPF_FLAG_NTAP_ON) && (flags & MPF_FLAG_NTAP_OFF)) return fail(MPF_ERR_ARG, "NTAP_ON with NTAP_OFF");
  if ((flags & MPF_FLAG_TC_PAIR) && (flags & MPF_FLAG_TC_SINGLE)) return fail(MPF_ERR_ARG, "TC_PAIR with TC_SINGLE");
  if ((flags & MPF_FLAG_HEAD_LOGITS_ON) && (flags & MPF_FLAG_HEAD_LOGITS_OFF))
    return fail(MPF_ERR_ARG, "HEAD_LOGITS_ON with HEAD_LOGITS_OFF");
  N->cfg.flags = flags;
  return MPF_OK;
}

mpf_status mpf_check(mpf_net* N, void* stream) {
  if (!N) return fail(MPF_ERR_ARG, "NULL net");
  cudaStream_t s = (cudaStream_t)stream;
  MPF_CUDA(cudaStreamSynchronize(s));
  MPF_CUDA(cudaGetLastError());
  if (N->bound) {
    int err = 0;
    MPF_CUDA(cudaMemcpy(&err, N->scratch + N->off_err, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) {
      MPF_CUDA(cudaMemset(N->scratch + N->off_err, 0, sizeof(int)));
      return fail(MPF_ERR_DATA, "a label >= classes (and != 255) was found; it was ignored");
    }
  }
  if (N->ex_on) {
    uint32_t t = 0;
    MPF_CUDA(cudaMemcpy(&t, N->ex_own + ExLayout::kTimeout, sizeof(t), cudaMemcpyDeviceToHost));
    if (t)
      return fail(MPF_ERR_INTERNAL, "gradient exchange: timed out waiting for rank " + std::to_string(t - 1) +
                                        "; parameters not updated");
  }
  return MPF_OK;
}

// ---------------------------------------------------------------- CUDA IPC (exchange buffers)
typedef CUresult (*PFN_getAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

mpf_status mpf_ipc_export(const void* d_ptr, void* handle64, uint64_t* offset) {
  if (!d_ptr || !handle64 || !offset) return fail(MPF_ERR_ARG, "NULL argument");
  static PFN_getAddressRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(MPF_ERR_CUDA, "cuMemGetAddressRange entry point not found");
    get_range = (PFN_getAddressRange)fn;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (CUdeviceptr)(uintptr_t)d_ptr) != CUDA_SUCCESS)
    return fail(MPF_ERR_CUDA, "cuMemGetAddressRange failed (not a device allocation?)");
  cudaIpcMemHandle_t h;
  MPF_CUDA(cudaIpcGetMemHandle(&h, (void*)(uintptr_t)base));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  memcpy(handle64, &h, sizeof(h));
  *offset = (uint64_t)((uintptr_t)d_ptr - (uintptr_t)base);
  return MPF_OK;
}

mpf_status mpf_ipc_open(const void* handle64, uint64_t offset, void** d_ptr) {
  if (!handle64 || !d_ptr) return fail(MPF_ERR_ARG, "NULL argument");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  void* base = nullptr;
  MPF_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
  *d_ptr = (char*)base + offset;
  return MPF_OK;
}

mpf_status mpf_ipc_close(void* d_ptr, uint64_t offset) {
  if (!d_ptr) return fail(MPF_ERR_ARG, "NULL argument");
  MPF_CUDA(cudaIpcCloseMemHandle((char*)d_ptr - offset));
  return MPF_OK;
}

}  // extern "C"
