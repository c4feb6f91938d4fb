/*
 * oracle/o1_patch.c — ORACLE O1: naive patch-by-patch MPCNN training, fp64, plain C.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this code.  The product path
 * (paper_1302_1690_b200/) never links, imports or calls it, and this file shares
 * no code, header, table or helper with the CUDA path.
 *
 * What it computes is the *plain definition* that the paper's whole-image method
 * reaches exactly (§2 "evaluate the net on every patch contained in
 * it"; §3.2 "every pixel is replaced by the output of the
 * corresponding MPCNN applied to every patch"; "trained on a
 * computationally expensive patch-by-patch basis").  For every selected output
 * pixel (y, x) of an image (reading R7: output (y,x) <-> the P x P patch with
 * top-left pixel (y,x)):
 *   1. take the P x P patch x[:, y:y+P, x:x+P];
 *   2. classical MPCNN forward (§2):
 *        C  : valid 2-D cross-correlation (R10), full connectivity between input
 *             and output maps, + bias, then tanh (R11)
 *        MP : non-overlapping k x k max; argmax = first occurrence
 *             in row-major scan (strict '>', R6); exact divisibility required in
 *             patch mode
 *        FC : affine map of the input vector, i.e. a k x k
 *             cross-correlation over the remaining k x k x C volume (R12), + tanh,
 *             except the last FC which is linear and feeds a softmax (R11, R15)
 *   3. multi-class cross-entropy per pixel ("MCCE ... each pixel
 *      independently"), class-weighted (R9): l = -w_t log p_t;
 *   4. classical per-patch back-propagation (PAPER.md:63 refers to the standard
 *      MPCNN backprop): dl/dlogits = w_t (p - onehot_t); tanh' = 1 - y^2 from
 *      the stored outputs; max-pool routes the delta to its argmax.
 * Per image it returns sum over the selected labelled pixels of l and of dl/dTheta
 * (the caller divides by the labelled count n_lab: R8), and the softmax
 * probabilities of every selected pixel.
 *
 * Parameter order: layer order; W[out][in][kr][kc]; then b[out].
 *
 * Pixels are split statically over n_threads POSIX threads; each thread keeps
 * its own gradient accumulator and they are summed in thread order, so results
 * are deterministic for a fixed thread count.  No blocking, caching, im2col or
 * reordering beyond the definition.
 */
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

#define O1_MAXL 32

enum { O1_CONV = 0, O1_POOL = 1, O1_FC = 2 };
enum { O1_TANH = 0, O1_IDENTITY = 1, O1_LOGISTIC = 2 };
enum { O1_OK = 0, O1_ERR_CONFIG = 2, O1_ERR_DATA = 3, O1_ERR_NOMEM = 6 };

typedef struct {
  int kind, k, n_out, act;
} o1_layer;

typedef struct {
  int n_layers, in_ch, P, classes;
  const o1_layer* L;
  int ch[O1_MAXL + 1]; /* channels of activation a[l]; a[0] is the patch */
  int sz[O1_MAXL + 1]; /* spatial size (square) of a[l] */
  long woff[O1_MAXL];  /* offset of W of layer l in the flat parameters */
  long boff[O1_MAXL];  /* offset of b */
  long n_params;
  long asz[O1_MAXL + 1]; /* elements of a[l] */
} net_t;

/* Shape chain in patch mode; returns O1_ERR_CONFIG when the layer list does not
 * reduce a P x P patch to 1 x 1 at the last layer. */
static int net_plan(net_t* n, const o1_layer* L, int n_layers, int in_ch, int P) {
  if (n_layers < 1 || n_layers > O1_MAXL || in_ch < 1 || P < 1) return O1_ERR_CONFIG;
  n->L = L;
  n->n_layers = n_layers;
  n->in_ch = in_ch;
  n->P = P;
  n->ch[0] = in_ch;
  n->sz[0] = P;
  long off = 0;
  for (int l = 0; l < n_layers; ++l) {
    const o1_layer* y = &L[l];
    if (y->k < 1) return O1_ERR_CONFIG;
    if (y->kind == O1_CONV || y->kind == O1_FC) {
      if (y->n_out < 1 || y->k > n->sz[l]) return O1_ERR_CONFIG;
      if (y->kind == O1_FC && y->k != n->sz[l]) return O1_ERR_CONFIG; /* FC sees the whole volume */
      n->ch[l + 1] = y->n_out;
      n->sz[l + 1] = n->sz[l] - y->k + 1;
      n->woff[l] = off;
      off += (long)y->n_out * n->ch[l] * y->k * y->k;
      n->boff[l] = off;
      off += y->n_out;
    } else if (y->kind == O1_POOL) {
      if (n->sz[l] % y->k != 0) return O1_ERR_CONFIG; /* exact divisibility in patch mode */
      n->ch[l + 1] = n->ch[l];
      n->sz[l + 1] = n->sz[l] / y->k;
      n->woff[l] = n->boff[l] = -1;
    } else {
      return O1_ERR_CONFIG;
    }
  }
  if (n->sz[n_layers] != 1) return O1_ERR_CONFIG;
  if (L[n_layers - 1].kind == O1_POOL || L[n_layers - 1].act != O1_IDENTITY) return O1_ERR_CONFIG;
  n->classes = n->ch[n_layers];
  n->n_params = off;
  for (int l = 0; l <= n_layers; ++l) n->asz[l] = (long)n->ch[l] * n->sz[l] * n->sz[l];
  return O1_OK;
}

static double act_f(int act, double v) {
  if (act == O1_TANH) return tanh(v);
  if (act == O1_LOGISTIC) return 1.0 / (1.0 + exp(-v));
  return v;
}

/* derivative of the activation from its output y */
static double act_d(int act, double y) {
  if (act == O1_TANH) return 1.0 - y * y;
  if (act == O1_LOGISTIC) return y * (1.0 - y);
  return 1.0;
}

typedef struct {
  const net_t* net;
  const double* params;
  const double* image;
  int H, W, O_H, O_W;
  const unsigned char* labels;
  const double* class_w;
  const int* pix;
  int n_pix;
  int p_begin, p_end;
  int want_grad;
  double* probs;
  /* per-thread results */
  double* grad;
  double loss;
  long n_lab;
  int status;
} job_t;

static void* run_job(void* arg) {
  job_t* J = (job_t*)arg;
  const net_t* N = J->net;
  const int NL = N->n_layers;
  const double* th = J->params;
  /* per-layer activation, delta and argmax buffers (patch-sized, reused) */
  double* a[O1_MAXL + 1];
  double* d[O1_MAXL + 1];
  int* am[O1_MAXL];
  int ok = 1;
  for (int l = 0; l <= NL; ++l) {
    a[l] = (double*)malloc(sizeof(double) * N->asz[l]);
    d[l] = (double*)malloc(sizeof(double) * N->asz[l]);
    if (!a[l] || !d[l]) ok = 0;
  }
  for (int l = 0; l < NL; ++l) {
    am[l] = (int*)malloc(sizeof(int) * (N->asz[l + 1] > 0 ? N->asz[l + 1] : 1));
    if (!am[l]) ok = 0;
  }
  if (!ok) {
    J->status = O1_ERR_NOMEM;
    return NULL;
  }
  const int C = N->classes;
  double* p = (double*)malloc(sizeof(double) * C);

  for (int q = J->p_begin; q < J->p_end; ++q) {
    const int lin = J->pix ? J->pix[q] : q;
    const int y0 = lin / J->O_W, x0 = lin % J->O_W;
    /* 1. the patch with top-left (y0, x0) */
    const int P = N->P;
    for (int c = 0; c < N->in_ch; ++c)
      for (int i = 0; i < P; ++i)
        for (int j = 0; j < P; ++j)
          a[0][((long)c * P + i) * P + j] = J->image[((long)c * J->H + y0 + i) * J->W + x0 + j];
    /* 2. forward */
    for (int l = 0; l < NL; ++l) {
      const o1_layer* Ly = &N->L[l];
      const int ci_n = N->ch[l], co_n = N->ch[l + 1], si = N->sz[l], so = N->sz[l + 1], k = Ly->k;
      if (Ly->kind == O1_POOL) {
        for (int c = 0; c < ci_n; ++c)
          for (int i = 0; i < so; ++i)
            for (int j = 0; j < so; ++j) {
              double best = a[l][((long)c * si + k * i) * si + k * j];
              int arg = 0;
              for (int dy = 0; dy < k; ++dy)
                for (int dx = 0; dx < k; ++dx) {
                  double v = a[l][((long)c * si + k * i + dy) * si + k * j + dx];
                  if (v > best) { best = v; arg = dy * k + dx; }
                }
              a[l + 1][((long)c * so + i) * so + j] = best;
              am[l][((long)c * so + i) * so + j] = arg;
            }
      } else {
        const double* Wt = th + N->woff[l];
        const double* b = th + N->boff[l];
        for (int co = 0; co < co_n; ++co)
          for (int i = 0; i < so; ++i)
            for (int j = 0; j < so; ++j) {
              double s = b[co];
              for (int ci = 0; ci < ci_n; ++ci)
                for (int ky = 0; ky < k; ++ky)
                  for (int kx = 0; kx < k; ++kx)
                    s += Wt[(((long)co * ci_n + ci) * k + ky) * k + kx] *
                         a[l][((long)ci * si + i + ky) * si + j + kx];
              a[l + 1][((long)co * so + i) * so + j] = act_f(Ly->act, s);
            }
      }
    }
    /* softmax over the C linear outputs */
    double mx = a[NL][0];
    for (int c = 1; c < C; ++c) if (a[NL][c] > mx) mx = a[NL][c];
    double z = 0.0;
    for (int c = 0; c < C; ++c) { p[c] = exp(a[NL][c] - mx); z += p[c]; }
    for (int c = 0; c < C; ++c) p[c] /= z;
    if (J->probs)
      for (int c = 0; c < C; ++c) J->probs[(long)q * C + c] = p[c];

    const unsigned char t = J->labels ? J->labels[lin] : 255;
    if (t == 255) continue; /* ignore label (R7/R8) */
    if (t >= C) { J->status = O1_ERR_DATA; continue; }
    const double w = J->class_w ? J->class_w[t] : 1.0;
    /* 3. MCCE */
    J->loss += -w * log(p[t]);
    J->n_lab += 1;
    if (!J->want_grad) continue;
    /* 4. backward: dl/dlogits = w (p - onehot) */
    for (int c = 0; c < C; ++c) d[NL][c] = w * (p[c] - (c == t ? 1.0 : 0.0));
    for (int l = NL - 1; l >= 0; --l) {
      const o1_layer* Ly = &N->L[l];
      const int ci_n = N->ch[l], co_n = N->ch[l + 1], si = N->sz[l], so = N->sz[l + 1], k = Ly->k;
      if (l > 0) memset(d[l], 0, sizeof(double) * N->asz[l]);
      if (Ly->kind == O1_POOL) {
        if (l == 0) continue; /* nothing upstream of the patch */
        for (int c = 0; c < ci_n; ++c)
          for (int i = 0; i < so; ++i)
            for (int j = 0; j < so; ++j) {
              int arg = am[l][((long)c * so + i) * so + j];
              int dy = arg / k, dx = arg % k;
              d[l][((long)c * si + k * i + dy) * si + k * j + dx] += d[l + 1][((long)c * so + i) * so + j];
            }
      } else {
        const double* Wt = th + N->woff[l];
        double* gW = J->grad + N->woff[l];
        double* gb = J->grad + N->boff[l];
        for (int co = 0; co < co_n; ++co)
          for (int i = 0; i < so; ++i)
            for (int j = 0; j < so; ++j) {
              const long o = ((long)co * so + i) * so + j;
              const double dp = d[l + 1][o] * act_d(Ly->act, a[l + 1][o]);
              gb[co] += dp;
              for (int ci = 0; ci < ci_n; ++ci)
                for (int ky = 0; ky < k; ++ky)
                  for (int kx = 0; kx < k; ++kx) {
                    const long wi = (((long)co * ci_n + ci) * k + ky) * k + kx;
                    const long ai = ((long)ci * si + i + ky) * si + j + kx;
                    gW[wi] += dp * a[l][ai];
                    if (l > 0) d[l][ai] += dp * Wt[wi];
                  }
            }
      }
    }
  }
  free(p);
  for (int l = 0; l <= NL; ++l) { free(a[l]); free(d[l]); }
  for (int l = 0; l < NL; ++l) free(am[l]);
  return NULL;
}

/* Number of parameters of a layer list (or -1 on a config error). */
long o1_n_params(const o1_layer* layers, int n_layers, int in_ch, int P) {
  net_t n;
  if (net_plan(&n, layers, n_layers, in_ch, P) != O1_OK) return -1;
  return n.n_params;
}

/*
 * One image.  image: [in_ch][H][W] fp64; labels: [O_H][O_W] (O = H-P+1) uint8,
 * 255 = ignore, may be NULL (forward only); class_w: [C] or NULL (= 1);
 * pix: linear output indices y*O_W + x to process, or NULL for all O_H*O_W.
 * grad_sum (+=, [n_params]) may be NULL for forward/loss only; probs: [n_pix][C]
 * or NULL.  Returns O1_OK, O1_ERR_CONFIG, O1_ERR_DATA (label >= C) or O1_ERR_NOMEM.
 */
int o1_image(const o1_layer* layers, int n_layers, int in_ch, int P, const double* params,
             const double* image, int H, int W, const unsigned char* labels, const double* class_w,
             const int* pix, int n_pix, int n_threads, double* grad_sum, double* loss_sum,
             long* n_lab, double* probs) {
  net_t N;
  int st = net_plan(&N, layers, n_layers, in_ch, P);
  if (st != O1_OK) return st;
  if (H < P || W < P) return O1_ERR_CONFIG;
  const int O_H = H - P + 1, O_W = W - P + 1;
  if (!pix) n_pix = O_H * O_W;
  if (n_threads < 1) n_threads = 1;
  if (n_threads > n_pix) n_threads = n_pix > 0 ? n_pix : 1;
  job_t* jobs = (job_t*)calloc(n_threads, sizeof(job_t));
  pthread_t* tid = (pthread_t*)calloc(n_threads, sizeof(pthread_t));
  if (!jobs || !tid) return O1_ERR_NOMEM;
  for (int t = 0; t < n_threads; ++t) {
    job_t* J = &jobs[t];
    J->net = &N;
    J->params = params;
    J->image = image;
    J->H = H; J->W = W; J->O_H = O_H; J->O_W = O_W;
    J->labels = labels;
    J->class_w = class_w;
    J->pix = pix;
    J->n_pix = n_pix;
    J->p_begin = (int)((long)n_pix * t / n_threads);
    J->p_end = (int)((long)n_pix * (t + 1) / n_threads);
    J->want_grad = grad_sum != NULL;
    J->probs = probs;
    J->grad = grad_sum ? (double*)calloc(N.n_params, sizeof(double)) : NULL;
    if (grad_sum && !J->grad) return O1_ERR_NOMEM;
  }
  for (int t = 1; t < n_threads; ++t) pthread_create(&tid[t], NULL, run_job, &jobs[t]);
  run_job(&jobs[0]);
  for (int t = 1; t < n_threads; ++t) pthread_join(tid[t], NULL);
  /* fixed-order reduction over threads */
  double loss = 0.0;
  long cnt = 0;
  st = O1_OK;
  for (int t = 0; t < n_threads; ++t) {
    if (jobs[t].status != O1_OK) st = jobs[t].status;
    loss += jobs[t].loss;
    cnt += jobs[t].n_lab;
    if (grad_sum) {
      for (long i = 0; i < N.n_params; ++i) grad_sum[i] += jobs[t].grad[i];
      free(jobs[t].grad);
    }
  }
  if (loss_sum) *loss_sum += loss;
  if (n_lab) *n_lab += cnt;
  free(jobs);
  free(tid);
  return st;
}
