/* TEST INFRASTRUCTURE — NOT PART OF THE PRODUCT.  See pbrl_oracle.h for the contract.
 *
 * A plain-C restatement of the reference population update.  Arithmetic follows the
 * reference operation by operation (same association, same float/double boundaries,
 * no FMA contraction: built with -ffp-contract=off), so results are bit-identical to the
 * reference built with its Release flags.  Each block cites the reference lines it restates.
 */
#include "pbrl_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define ORA_MAXL 8
enum { ACT_NONE = 0, ACT_RELU = 1, ACT_TANH = 2 };
enum { USE_INIT_W = 1, USE_INIT_B = 2, USE_EXPLORE = 3, USE_TARGET_NOISE = 4, USE_SAC_EPS = 5,
       USE_SAC_EPS_T = 6, USE_SAMPLE = 7, USE_DONOR = 8, USE_HYPER = 9, USE_GENERIC = 12 };

/* ------------------------------------------------------------------ RNG (rng.hpp:13-95) */
uint64_t ora_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

uint64_t ora_stream_key(uint64_t seed, uint64_t stream, uint64_t use, uint64_t step) {
  uint64_t k = ora_mix64(seed);
  k = ora_mix64(k ^ stream);
  k = ora_mix64(k ^ use);
  return ora_mix64(k ^ step);
}

uint64_t ora_bits(uint64_t key, uint64_t c) { return ora_mix64(key ^ ora_mix64(c)); }

double ora_uniform(uint64_t key, uint64_t c) {
  return (double)(ora_bits(key, c) >> 11) * 0x1.0p-53;
}

static double uniform_pos(uint64_t key, uint64_t c) {
  return ((double)(ora_bits(key, c) >> 11) + 1.0) * 0x1.0p-53;
}

static double uniform_in(uint64_t key, uint64_t c, double lo, double hi) {
  return lo + (hi - lo) * ora_uniform(key, c);
}

double ora_normal_pair(uint64_t key, uint64_t c) {
  const double u1 = uniform_pos(key, c);
  const double u2 = ora_uniform(key, c + 1);
  return sqrt(-2.0 * log(u1)) * cos(6.28318530717958647692 * u2);
}

/* RngSequence (rng.hpp:74-95) as (key, *next) */
static uint64_t seq_bits(uint64_t key, uint64_t* next) { return ora_bits(key, (*next)++); }
static double seq_uniform(uint64_t key, uint64_t* next, double lo, double hi) {
  return uniform_in(key, (*next)++, lo, hi);
}
static double seq_log_uniform(uint64_t key, uint64_t* next, double lo, double hi) {
  return exp(seq_uniform(key, next, log(lo), log(hi)));
}

/* std::clamp / std::min / std::max with the libstdc++ comparison order */
static float clampf_(float v, float lo, float hi) { return v < lo ? lo : (hi < v ? hi : v); }
static float minf_(float a, float b) { return b < a ? b : a; }
static float maxf_(float a, float b) { return a < b ? b : a; }

/* ------------------------------------------------------------------ MLP (net_pop.hpp) */
typedef struct {
  int depth;
  uint64_t dims[ORA_MAXL + 1];
  int out_act;
  float out_scale;
  uint64_t P;
  uint64_t woff[ORA_MAXL], boff[ORA_MAXL];
} ora_net;

static void net_make(ora_net* nt, const uint64_t* dims, int ndims, int out_act, float scale) {
  memset(nt, 0, sizeof(*nt));
  nt->depth = ndims - 1;
  nt->out_act = out_act;
  nt->out_scale = scale;
  uint64_t at = 0;
  for (int i = 0; i < ndims; ++i) nt->dims[i] = dims[i];
  for (int l = 0; l < nt->depth; ++l) {
    nt->woff[l] = at;
    at += dims[l] * dims[l + 1];
    nt->boff[l] = at;
    at += dims[l + 1];
  }
  nt->P = at;
}

/* init_pop_mlp, net_pop.hpp:69-100 */
static void net_init(const ora_net* nt, float* p, uint64_t n, uint64_t seed) {
  for (int l = 0; l < nt->depth; ++l) {
    const uint64_t fi = nt->dims[l], fo = nt->dims[l + 1];
    const double wb = sqrt(1.0 / (double)fi);
    const double bb = 1.0 / sqrt((double)fi);
    for (uint64_t m = 0; m < n; ++m) {
      const uint64_t ws = ora_stream_key(seed, m, USE_INIT_W, (uint64_t)l);
      const uint64_t bs = ora_stream_key(seed, m, USE_INIT_B, (uint64_t)l);
      float* w = p + m * nt->P + nt->woff[l];
      float* b = p + m * nt->P + nt->boff[l];
      for (uint64_t e = 0; e < fi * fo; ++e) w[e] = (float)uniform_in(ws, e, -wb, wb);
      for (uint64_t e = 0; e < fo; ++e) b[e] = (float)uniform_in(bs, e, -bb, bb);
    }
  }
}

/* ForwardCache, net_pop.hpp:103-107: each layer's input and pre-activation */
typedef struct {
  uint64_t n, rows;
  int depth;
  float* in[ORA_MAXL];
  float* z[ORA_MAXL];
  float* out;
} ora_cache;

static void cache_free(ora_cache* c) {
  for (int l = 0; l < c->depth; ++l) {
    free(c->in[l]);
    free(c->z[l]);
  }
  free(c->out);
  memset(c, 0, sizeof(*c));
}

/* Tensor-core operand emulation (NOT the reference: used only by oracle/derive_tolerances.py to
 * derive the TF32 / BF16 parity tolerances).  0 = exact fp32 (the reference arithmetic), 1 = TF32
 * operands (fp32 with the low 13 mantissa bits dropped, as tcgen05 kind::tf32 reads fp32 data),
 * 2 = BF16 operands (round to nearest even).  Applied to both operands of every hidden-layer
 * product -- forward, dX and dW -- i.e. exactly the products the library runs on tcgen05; the
 * output layers, biases, losses, Adam and Polyak stay fp32 as in the library. */
static int g_emul = 0;
void ora_set_emulation(int mode) { g_emul = mode; }

static float emu(float x) {
  uint32_t u;
  memcpy(&u, &x, 4);
  if (g_emul == 1) {
    u &= 0xffffe000u;
  } else if (g_emul == 2) {
    if ((u & 0x7fffffffu) > 0x7f800000u) return x;
    u = (u + 0x7fffu + ((u >> 16) & 1u)) & 0xffff0000u;
  } else {
    return x;
  }
  memcpy(&x, &u, 4);
  return x;
}

/* rounded copy of count floats (malloc'd), or NULL when emulation is off / not a TC product */
static float* emu_copy(const float* x, uint64_t count, int tc) {
  if (!g_emul || !tc) return NULL;
  float* o = (float*)malloc(sizeof(float) * count);
  for (uint64_t i = 0; i < count; ++i) o[i] = emu(x[i]);
  return o;
}


/* Members are independent, so the per-member loops of the MLP forward and
 * backward run on a few pthreads; each member's arithmetic is unchanged, so the result bits do
 * not depend on the thread count (ORA_THREADS, default: online CPUs, at most 32). */
typedef void (*member_fn)(void* ctx, uint64_t m);
typedef struct {
  member_fn fn;
  void* ctx;
  uint64_t n, stride, first;
} par_job;

static void* par_worker(void* arg) {
  par_job* j = (par_job*)arg;
  for (uint64_t m = j->first; m < j->n; m += j->stride) j->fn(j->ctx, m);
  return NULL;
}

static void for_members(uint64_t n, member_fn fn, void* ctx) {
  static long threads = 0;
  if (threads == 0) {
    const char* e = getenv("ORA_THREADS");
    threads = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
    if (threads < 1) threads = 1;
    if (threads > 32) threads = 32;
  }
  uint64_t t = (uint64_t)threads < n ? (uint64_t)threads : n;
  if (t <= 1) {
    for (uint64_t m = 0; m < n; ++m) fn(ctx, m);
    return;
  }
  pthread_t tid[32];
  par_job job[32];
  for (uint64_t i = 0; i < t; ++i) {
    job[i] = (par_job){fn, ctx, n, t, i};
    pthread_create(&tid[i], NULL, par_worker, &job[i]);
  }
  for (uint64_t i = 0; i < t; ++i) pthread_join(tid[i], NULL);
}

/* pop_matmul (pop_tensor.hpp:139-170) + pop_add_bias (:213-232) for one member */
static void layer_forward(const float* x, uint64_t rows, uint64_t in, const float* w,
                          const float* bias, uint64_t out, float* z, int tc) {
  float* xe = emu_copy(x, rows * in, tc);
  float* we = emu_copy(w, in * out, tc);
  if (xe) x = xe;
  if (we) w = we;
  for (uint64_t r = 0; r < rows; ++r) {
    const float* xr = x + r * in;
    float* zr = z + r * out;
    const float x0 = xr[0];
    for (uint64_t o = 0; o < out; ++o) zr[o] = x0 * w[o];
    for (uint64_t i = 1; i < in; ++i) {
      const float xi = xr[i];
      const float* wr = w + i * out;
      for (uint64_t o = 0; o < out; ++o) zr[o] += xi * wr[o];
    }
    for (uint64_t o = 0; o < out; ++o) zr[o] = zr[o] + bias[o];
  }
  free(xe);
  free(we);
}

/* activation (pop_tensor.hpp:254-271) */
static void act_forward(const float* z, float* y, uint64_t count, int act) {
  for (uint64_t i = 0; i < count; ++i) {
    if (act == ACT_RELU) y[i] = z[i] > 0.0f ? z[i] : 0.0f;
    else if (act == ACT_TANH) y[i] = tanhf(z[i]);
    else y[i] = z[i];
  }
}

typedef struct {
  const ora_net* nt;
  const float* params;
  ora_cache* c;
  uint64_t rows;
  int l;
} fwd_ctx;

static void fwd_member(void* p, uint64_t m) {
  const fwd_ctx* f = (const fwd_ctx*)p;
  const ora_net* nt = f->nt;
  const uint64_t in = nt->dims[f->l], out = nt->dims[f->l + 1], rows = f->rows;
  layer_forward(f->c->in[f->l] + m * rows * in, rows, in, f->params + m * nt->P + nt->woff[f->l],
                f->params + m * nt->P + nt->boff[f->l], out, f->c->z[f->l] + m * rows * out,
                f->l + 1 < nt->depth);
}

/* pop_mlp_forward, net_pop.hpp:109-131 */
static void mlp_forward(const ora_net* nt, const float* params, uint64_t n, uint64_t rows,
                        const float* x, ora_cache* c) {
  memset(c, 0, sizeof(*c));
  c->n = n;
  c->rows = rows;
  c->depth = nt->depth;
  c->in[0] = (float*)malloc(sizeof(float) * n * rows * nt->dims[0]);
  memcpy(c->in[0], x, sizeof(float) * n * rows * nt->dims[0]);
  for (int l = 0; l < nt->depth; ++l) {
    const uint64_t in = nt->dims[l], out = nt->dims[l + 1];
    c->z[l] = (float*)malloc(sizeof(float) * n * rows * out);
    fwd_ctx fc = {nt, params, c, rows, l};
    for_members(n, fwd_member, &fc);
    float* y = (float*)malloc(sizeof(float) * n * rows * out);
    act_forward(c->z[l], y, n * rows * out, (l + 1 < nt->depth) ? ACT_RELU : nt->out_act);
    if (l + 1 < nt->depth) c->in[l + 1] = y;
    else c->out = y;
  }
  if (nt->out_scale != 1.0f) {
    const uint64_t cnt = n * rows * nt->dims[nt->depth];
    for (uint64_t i = 0; i < cnt; ++i) c->out[i] *= nt->out_scale;
  }
}

/* pop_mlp_backward, net_pop.hpp:134-160, composed of activation_backward
 * (pop_tensor.hpp:275-297), pop_add_bias_backward (:236-250) and pop_matmul_backward
 * (:173-210).  grads: [n][P] (overwritten); grad_x: [n][rows][dims[0]] or NULL. */
typedef struct {
  const ora_net* nt;
  const float* params;
  const ora_cache* c;
  const float* grad_y;
  float* grads;
  float* grad_x;
  uint64_t widest;
} bwd_ctx;

static void bwd_member(void* p, uint64_t m) {
  const bwd_ctx* f = (const bwd_ctx*)p;
  const ora_net* nt = f->nt;
  const float* params = f->params;
  const ora_cache* c = f->c;
  const float* grad_y = f->grad_y;
  float* grads = f->grads;
  float* grad_x = f->grad_x;
  const uint64_t rows = c->rows, widest = f->widest;
  float* g = (float*)malloc(sizeof(float) * rows * widest);
  float* gx = (float*)malloc(sizeof(float) * rows * widest);
  const uint64_t dout = nt->dims[nt->depth];
  memcpy(g, grad_y + m * rows * dout, sizeof(float) * rows * dout);
  if (nt->out_scale != 1.0f) {
    for (uint64_t i = 0; i < rows * dout; ++i) g[i] *= nt->out_scale;
  }
  for (int l = nt->depth - 1; l >= 0; --l) {
    const uint64_t in = nt->dims[l], out = nt->dims[l + 1];
    const int act = (l + 1 < nt->depth) ? ACT_RELU : nt->out_act;
    const float* z = c->z[l] + m * rows * out;
    if (act == ACT_RELU) {
      for (uint64_t i = 0; i < rows * out; ++i) {
        if (!(z[i] > 0.0f)) g[i] = 0.0f;
      }
    } else if (act == ACT_TANH) {
      for (uint64_t i = 0; i < rows * out; ++i) {
        const float t = tanhf(z[i]);
        g[i] *= (1.0f - t * t);
      }
    }
    /* emulation only: the hidden-layer cotangent is a tensor-core operand */
    const int tc = l + 1 < nt->depth;
    if (g_emul && tc) {
      for (uint64_t i = 0; i < rows * out; ++i) g[i] = emu(g[i]);
    }
    float* gb = grads + m * nt->P + nt->boff[l];
    for (uint64_t o = 0; o < out; ++o) gb[o] = 0.0f;
    for (uint64_t r = 0; r < rows; ++r) {
      for (uint64_t o = 0; o < out; ++o) gb[o] += g[r * out + o];
    }
    const float* w = params + m * nt->P + nt->woff[l];
    float* gw = grads + m * nt->P + nt->woff[l];
    const float* x = c->in[l] + m * rows * in;
    float* we = emu_copy(w, in * out, tc);
    float* xe = emu_copy(x, rows * in, tc);
    if (we) w = we;
    if (xe) x = xe;
    for (uint64_t i = 0; i < in * out; ++i) gw[i] = 0.0f;
    for (uint64_t r = 0; r < rows; ++r) {
      const float* gr = g + r * out;
      const float* xr = x + r * in;
      for (uint64_t i = 0; i < in; ++i) {
        const float* wr = w + i * out;
        float acc = 0.0f;
        for (uint64_t o = 0; o < out; ++o) acc += gr[o] * wr[o];
        gx[r * in + i] = acc;
        const float xi = xr[i];
        float* gwr = gw + i * out;
        for (uint64_t o = 0; o < out; ++o) gwr[o] += xi * gr[o];
      }
    }
    free(we);
    free(xe);
    float* tmp = g;
    g = gx;
    gx = tmp;
  }
  if (grad_x) memcpy(grad_x + m * rows * nt->dims[0], g, sizeof(float) * rows * nt->dims[0]);
  free(g);
  free(gx);
}

static void mlp_backward(const ora_net* nt, const float* params, const ora_cache* c,
                         const float* grad_y, float* grads, float* grad_x) {
  uint64_t widest = 0;
  for (int l = 0; l <= nt->depth; ++l) widest = nt->dims[l] > widest ? nt->dims[l] : widest;
  bwd_ctx bc = {nt, params, c, grad_y, grads, grad_x, widest};
  for_members(c->n, bwd_member, &bc);
}

/* adam_step_inplace for one member (pop_tensor.hpp:328-366); t is shared by every tensor of the
 * network because MlpAdam::step (optim.hpp:23-30) steps them together under one mask. */
static void adam_member(float* p, const float* g, float* mo, float* vo, int64_t* t, uint64_t P,
                        double lr) {
  *t += 1;
  const float b1 = (float)0.9;
  const float b2 = (float)0.999;
  const float corr1 = (float)(1.0 - pow(0.9, (double)*t));
  const float corr2 = (float)(1.0 - pow(0.999, (double)*t));
  const float step = (float)lr;
  const float epsv = (float)1e-8;
  for (uint64_t k = 0; k < P; ++k) {
    mo[k] = b1 * mo[k] + (1.0f - b1) * g[k];
    vo[k] = b2 * vo[k] + (1.0f - b2) * g[k] * g[k];
    const float mhat = mo[k] / corr1;
    const float vhat = vo[k] / corr2;
    p[k] -= step * mhat / (sqrtf(vhat) + epsv);
  }
}

/* soft_update_members_inplace, one member (pop_tensor.hpp:412-428) */
static void polyak_member(float* tg, const float* on, uint64_t P, double tau) {
  const float a = (float)tau;
  const float b = (float)(1.0 - tau);
  for (uint64_t k = 0; k < P; ++k) tg[k] = a * on[k] + b * tg[k];
}

/* concat_features (pop_tensor.hpp:432-456) */
static float* concat(const float* x, const float* y, uint64_t n, uint64_t rows, uint64_t fx,
                     uint64_t fy) {
  float* o = (float*)malloc(sizeof(float) * n * rows * (fx + fy));
  for (uint64_t i = 0; i < n * rows; ++i) {
    memcpy(o + i * (fx + fy), x + i * fx, sizeof(float) * fx);
    memcpy(o + i * (fx + fy) + fx, y + i * fy, sizeof(float) * fy);
  }
  return o;
}

/* columns [from, from+cnt) of a [rows][f] block (split_features, pop_tensor.hpp:460-477) */
static float* take_cols(const float* x, uint64_t count, uint64_t f, uint64_t from, uint64_t cnt) {
  float* o = (float*)malloc(sizeof(float) * count * cnt);
  for (uint64_t i = 0; i < count; ++i) memcpy(o + i * cnt, x + i * f + from, sizeof(float) * cnt);
  return o;
}

/* mse_loss_grads, algos.hpp:288-314: per-member mean squared error and the full backward */
static void mse_grads(const ora_net* nt, const float* params, uint64_t n, uint64_t rows,
                      const float* input, const float* target, float* grads, double* loss) {
  ora_cache c;
  mlp_forward(nt, params, n, rows, input, &c);
  float* gq = (float*)malloc(sizeof(float) * n * rows);
  const float scale = 2.0f / (float)rows;
  for (uint64_t m = 0; m < n; ++m) {
    double acc = 0.0;
    for (uint64_t b = 0; b < rows; ++b) {
      const float dlt = c.out[m * rows + b] - target[m * rows + b];
      acc += (double)dlt * (double)dlt;
      gq[m * rows + b] = scale * dlt;
    }
    if (loss) loss[m] = acc / (double)rows;
  }
  mlp_backward(nt, params, &c, gq, grads, NULL);
  free(gq);
  cache_free(&c);
}

/* ------------------------------------------------------------------ TD3 (algos.hpp) */
struct ora_td3 {
  uint64_t n, ds, da;
  uint64_t nc;  /* critic population: n, or 1 in shared-critic mode (algos.hpp:197) */
  int shared;   /* PopMode::kSharedCritic */
  ora_net pol, cri;
  float bound;
  uint64_t seed;
  float* net[6];
  float* am[3];
  float* av[3];
  int64_t* at[3];
  double* delay_acc;
  uint64_t* steps;
  uint64_t* streams;
};

static const ora_net* td3_shape(const ora_td3* st, int net) {
  return (net <= 1) ? &st->pol : &st->cri;
}

static int td3_opt_index(int net) { return net == 0 ? 0 : (net == 2 ? 1 : 2); }

/* make_td3_state, algos.hpp:181-212; shared != 0 is PopMode::kSharedCritic (critic_n = 1) */
ora_td3* ora_td3_create_mode(uint64_t n, uint64_t ds, uint64_t da, const uint64_t* hidden,
                             uint32_t nh, double bound, uint64_t seed, int shared) {
  ora_td3* st = (ora_td3*)calloc(1, sizeof(ora_td3));
  st->n = n;
  st->shared = shared ? 1 : 0;
  st->nc = shared ? 1 : n;
  st->ds = ds;
  st->da = da;
  st->bound = (float)bound;
  st->seed = seed;
  uint64_t dims[ORA_MAXL + 1];
  dims[0] = ds;
  for (uint32_t i = 0; i < nh; ++i) dims[i + 1] = hidden[i];
  dims[nh + 1] = da;
  net_make(&st->pol, dims, (int)nh + 2, ACT_TANH, st->bound);
  dims[0] = ds + da;
  dims[nh + 1] = 1;
  net_make(&st->cri, dims, (int)nh + 2, ACT_NONE, 1.0f);
  const uint64_t nc = st->nc;
  for (int k = 0; k < 6; ++k) {
    st->net[k] = (float*)calloc((k <= 1 ? n : nc) * td3_shape(st, k)->P, sizeof(float));
  }
  net_init(&st->pol, st->net[0], n, ora_mix64(seed ^ 0xA1));
  net_init(&st->cri, st->net[2], nc, ora_mix64(seed ^ 0xB2));
  net_init(&st->cri, st->net[3], nc, ora_mix64(seed ^ 0xC3));
  memcpy(st->net[1], st->net[0], sizeof(float) * n * st->pol.P);
  memcpy(st->net[4], st->net[2], sizeof(float) * nc * st->cri.P);
  memcpy(st->net[5], st->net[3], sizeof(float) * nc * st->cri.P);
  for (int k = 0; k < 3; ++k) {
    const uint64_t P = (k == 0) ? st->pol.P : st->cri.P;
    const uint64_t cnt = (k == 0) ? n : nc;
    st->am[k] = (float*)calloc(cnt * P, sizeof(float));
    st->av[k] = (float*)calloc(cnt * P, sizeof(float));
    st->at[k] = (int64_t*)calloc(cnt, sizeof(int64_t));
  }
  st->delay_acc = (double*)calloc(n, sizeof(double));
  st->steps = (uint64_t*)calloc(n, sizeof(uint64_t));
  st->streams = (uint64_t*)calloc(n, sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) st->streams[i] = i;
  return st;
}

ora_td3* ora_td3_create(uint64_t n, uint64_t ds, uint64_t da, const uint64_t* hidden,
                        uint32_t nh, double bound, uint64_t seed) {
  return ora_td3_create_mode(n, ds, da, hidden, nh, bound, seed, 0);
}

void ora_td3_destroy(ora_td3* st) {
  if (!st) return;
  for (int k = 0; k < 6; ++k) free(st->net[k]);
  for (int k = 0; k < 3; ++k) {
    free(st->am[k]);
    free(st->av[k]);
    free(st->at[k]);
  }
  free(st->delay_acc);
  free(st->steps);
  free(st->streams);
  free(st);
}

uint64_t ora_td3_param_count(const ora_td3* st, int net) { return td3_shape(st, net)->P; }

void ora_td3_get_net(const ora_td3* st, int net, uint64_t m, float* out) {
  const uint64_t P = td3_shape(st, net)->P;
  memcpy(out, st->net[net] + m * P, sizeof(float) * P);
}

void ora_td3_set_net(ora_td3* st, int net, uint64_t m, const float* in) {
  const uint64_t P = td3_shape(st, net)->P;
  memcpy(st->net[net] + m * P, in, sizeof(float) * P);
}

void ora_td3_get_adam(const ora_td3* st, int net, uint64_t m, float* mo, float* vo, int64_t* t) {
  const int k = td3_opt_index(net);
  const uint64_t P = td3_shape(st, net)->P;
  memcpy(mo, st->am[k] + m * P, sizeof(float) * P);
  memcpy(vo, st->av[k] + m * P, sizeof(float) * P);
  *t = st->at[k][m];
}

void ora_td3_get_counters(const ora_td3* st, double* delay_acc, uint64_t* steps) {
  memcpy(delay_acc, st->delay_acc, sizeof(double) * st->n);
  memcpy(steps, st->steps, sizeof(uint64_t) * st->n);
}

#define HY(h, field, n, m) ((h)[(field) * (n) + (m)])
enum { TH_CLR = 0, TH_PLR, TH_DELAY, TH_EXPLORE, TH_TSTD, TH_TCLIP, TH_GAMMA, TH_TAU };

/* Td3Hyper::validate, algos.hpp:81-108 */
static int td3_validate(const double* h, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    if (!(HY(h, TH_CLR, n, i) > 0) || !(HY(h, TH_PLR, n, i) > 0)) return -2;
    const double dr = HY(h, TH_DELAY, n, i);
    if (!(dr > 0 && dr <= 1.0)) return -2;
    if (HY(h, TH_EXPLORE, n, i) < 0 || HY(h, TH_TSTD, n, i) < 0 || HY(h, TH_TCLIP, n, i) < 0)
      return -2;
    const double g = HY(h, TH_GAMMA, n, i);
    if (!(g >= 0.9 && g <= 1.0) && g != 0.0) return -2;
    const double tau = HY(h, TH_TAU, n, i);
    if (!(tau > 0 && tau <= 1.0)) return -2;
  }
  return 0;
}

/* td3_critic_target, algos.hpp:241-282 */
void ora_td3_target(const ora_td3* st, const float* s2, const float* r, const float* d,
                    uint64_t b, const double* hyper, float* y) {
  const uint64_t n = st->n, ds = st->ds, da = st->da;
  const float bound = st->bound;
  ora_cache cp;
  mlp_forward(&st->pol, st->net[1], n, b, s2, &cp);
  float* a2 = cp.out;
  for (uint64_t m = 0; m < n; ++m) {
    const uint64_t key = ora_stream_key(st->seed, st->streams[m], USE_TARGET_NOISE, st->steps[m]);
    const float sd = (float)(HY(hyper, TH_TSTD, n, m) * (double)bound);
    const float clip = (float)(HY(hyper, TH_TCLIP, n, m) * (double)bound);
    float* am = a2 + m * b * da;
    for (uint64_t e = 0; e < b * da; ++e) {
      float eps = (float)ora_normal_pair(key, 2 * e) * sd;
      eps = clampf_(eps, -clip, clip);
      am[e] = clampf_(am[e] + eps, -bound, bound);
    }
  }
  float* sa2 = concat(s2, a2, n, b, ds, da);
  ora_cache c1, c2;
  /* critic_forward (algos.hpp:219-227): a shared critic sees the population folded into its
   * batch axis -- the same row-major buffer read as nc = 1 member of n*b rows */
  const uint64_t rc = st->shared ? n * b : b;
  mlp_forward(&st->cri, st->net[4], st->nc, rc, sa2, &c1);
  mlp_forward(&st->cri, st->net[5], st->nc, rc, sa2, &c2);
  for (uint64_t m = 0; m < n; ++m) {
    const float g = (float)HY(hyper, TH_GAMMA, n, m);
    for (uint64_t i = 0; i < b; ++i) {
      const uint64_t k = m * b + i;
      const float qmin = minf_(c1.out[k], c2.out[k]);
      y[k] = r[k] + g * (1.0f - d[k]) * qmin;
    }
  }
  free(sa2);
  cache_free(&cp);
  cache_free(&c1);
  cache_free(&c2);
}

/* ------------------------------------------------------------------ DvD (evolve.hpp:304-525) */
double ora_dvd_lambda(uint64_t step, double start, double end, uint64_t horizon) {
  if (horizon == 0 || step >= horizon) return end;
  const double frac = (double)step / (double)horizon;
  return start + (end - start) * frac;
}

/* canonical_order (evolve.hpp:391-405): stable lexicographic sort of the embedding rows */
static const double* g_canon_e;
static uint64_t g_canon_dim;
static int canon_cmp(const void* pa, const void* pb) {
  const uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
  const double* ra = g_canon_e + a * g_canon_dim;
  const double* rb = g_canon_e + b * g_canon_dim;
  for (uint64_t k = 0; k < g_canon_dim; ++k) {
    if (ra[k] != rb[k]) return ra[k] < rb[k] ? -1 : 1;
  }
  return a < b ? -1 : (a > b ? 1 : 0); /* stable: ties keep index order */
}

/* cholesky / cholesky_inverse (evolve.hpp:364-400) */
static int chol(double* a, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) {
    for (uint64_t j = 0; j <= i; ++j) {
      double sum = a[i * n + j];
      for (uint64_t k = 0; k < j; ++k) sum -= a[i * n + k] * a[j * n + k];
      if (i == j) {
        if (!(sum > 0.0)) return 0;
        a[i * n + i] = sqrt(sum);
      } else {
        a[i * n + j] = sum / a[j * n + j];
      }
    }
    for (uint64_t j = i + 1; j < n; ++j) a[i * n + j] = 0.0;
  }
  return 1;
}

static void chol_inverse(const double* l, uint64_t n, double* inv) {
  double* col = (double*)malloc(sizeof(double) * n);
  for (uint64_t c = 0; c < n; ++c) {
    for (uint64_t i = 0; i < n; ++i) {
      double sum = (i == c) ? 1.0 : 0.0;
      for (uint64_t k = 0; k < i; ++k) sum -= l[i * n + k] * col[k];
      col[i] = sum / l[i * n + i];
    }
    for (uint64_t ii = n; ii-- > 0;) {
      double sum = col[ii];
      for (uint64_t k = ii + 1; k < n; ++k) sum -= l[k * n + ii] * col[k];
      col[ii] = sum / l[ii * n + ii];
    }
    for (uint64_t i = 0; i < n; ++i) inv[i * n + c] = col[i];
  }
  free(col);
}

/* dvd_loss, evolve.hpp:411-465 */
int ora_dvd_loss(const double* emb, uint64_t n, uint64_t dim, double length_scale, double jitter,
                 double lambda, double* loss, double* logdet_out, double* grad) {
  if (n < 2) return -2;
  if (!(length_scale > 0)) return -2;
  uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * n);
  for (uint64_t i = 0; i < n; ++i) order[i] = i;
  g_canon_e = emb;
  g_canon_dim = dim;
  qsort(order, n, sizeof(uint64_t), canon_cmp);
  const double inv2l2 = 1.0 / (2.0 * length_scale * length_scale);
  double* kernel = (double*)malloc(sizeof(double) * n * n);
  for (uint64_t i = 0; i < n; ++i) {
    kernel[i * n + i] = 1.0;
    const double* ri = emb + order[i] * dim;
    for (uint64_t j = 0; j < i; ++j) {
      const double* rj = emb + order[j] * dim;
      double d2 = 0;
      for (uint64_t k = 0; k < dim; ++k) {
        const double d = ri[k] - rj[k];
        d2 += d * d;
      }
      const double kij = exp(-d2 * inv2l2);
      kernel[i * n + j] = kij;
      kernel[j * n + i] = kij;
    }
  }
  double* m = (double*)malloc(sizeof(double) * n * n);
  memcpy(m, kernel, sizeof(double) * n * n);
  for (uint64_t i = 0; i < n; ++i) m[i * n + i] += jitter;
  if (!chol(m, n)) {
    free(order);
    free(kernel);
    free(m);
    return -10; /* DegeneratePopulationError */
  }
  double logdet = 0;
  for (uint64_t i = 0; i < n; ++i) logdet += 2.0 * log(m[i * n + i]);
  double* minv = (double*)malloc(sizeof(double) * n * n);
  chol_inverse(m, n, minv);
  if (logdet_out) *logdet_out = logdet;
  if (loss) *loss = -lambda * logdet;
  if (grad) {
    memset(grad, 0, sizeof(double) * n * dim);
    const double coef = 2.0 * lambda / (length_scale * length_scale);
    for (uint64_t i = 0; i < n; ++i) {
      double* gi = grad + order[i] * dim;
      const double* ri = emb + order[i] * dim;
      for (uint64_t j = 0; j < n; ++j) {
        if (j == i) continue;
        const double* rj = emb + order[j] * dim;
        const double w = coef * minv[i * n + j] * kernel[i * n + j];
        for (uint64_t k = 0; k < dim; ++k) gi[k] += w * (ri[k] - rj[k]);
      }
    }
  }
  free(order);
  free(kernel);
  free(m);
  free(minv);
  return 0;
}

static int dbl_cmp(const void* a, const void* b) {
  const double x = *(const double*)a, y = *(const double*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

/* median_pairwise_distance, evolve.hpp:469-486 */
double ora_median_pairwise_distance(const double* emb, uint64_t n, uint64_t dim) {
  if (n < 2) return 1.0;
  const uint64_t cnt = n * (n - 1) / 2;
  double* d = (double*)malloc(sizeof(double) * cnt);
  uint64_t at = 0;
  for (uint64_t i = 0; i < n; ++i) {
    for (uint64_t j = i + 1; j < n; ++j) {
      double d2 = 0;
      for (uint64_t k = 0; k < dim; ++k) {
        const double x = emb[i * dim + k] - emb[j * dim + k];
        d2 += x * x;
      }
      d[at++] = sqrt(d2);
    }
  }
  qsort(d, cnt, sizeof(double), dbl_cmp);
  const double med = d[cnt / 2];
  free(d);
  return med > 0 ? med : 1.0;
}

/* dvd_embed_cached (evolve.hpp:319-335): the probe states (double, cast to T as in
 * dvd_policy_hook) replicated per member, then the policy forward; out [n][m_states*da] */
static float* dvd_probe_block(const ora_td3* st, const double* probe, uint64_t ms) {
  float* x = (float*)malloc(sizeof(float) * st->n * ms * st->ds);
  for (uint64_t m = 0; m < st->n; ++m) {
    for (uint64_t i = 0; i < ms * st->ds; ++i) x[m * ms * st->ds + i] = (float)probe[i];
  }
  return x;
}

void ora_td3_dvd_embed(const ora_td3* st, const double* probe, uint64_t m_states, float* out) {
  float* x = dvd_probe_block(st, probe, m_states);
  ora_cache c;
  mlp_forward(&st->pol, st->net[0], st->n, m_states, x, &c);
  memcpy(out, c.out, sizeof(float) * st->n * m_states * st->da);
  cache_free(&c);
  free(x);
}

/* dvd_policy_hook (evolve.hpp:507-525) applied to the policy gradients g [n][Pp] */
static int dvd_hook(const ora_td3* st, const ora_dvd* dv, float* g) {
  if (dv->lambda == 0.0) return 0;
  const uint64_t n = st->n, ms = dv->m_states, da = st->da, dim = ms * da, Pp = st->pol.P;
  float* x = dvd_probe_block(st, dv->probe, ms);
  ora_cache c;
  mlp_forward(&st->pol, st->net[0], n, ms, x, &c);
  double* e = (double*)malloc(sizeof(double) * n * dim);
  double* ge = (double*)malloc(sizeof(double) * n * dim);
  for (uint64_t i = 0; i < n * dim; ++i) e[i] = (double)c.out[i];
  const int rc = ora_dvd_loss(e, n, dim, dv->length_scale, dv->jitter, dv->lambda, NULL, NULL, ge);
  if (rc == 0) {
    float* gf = (float*)malloc(sizeof(float) * n * dim);
    for (uint64_t i = 0; i < n * dim; ++i) gf[i] = (float)ge[i];
    float* dg = (float*)malloc(sizeof(float) * n * Pp);
    mlp_backward(&st->pol, st->net[0], &c, gf, dg, NULL);
    for (uint64_t i = 0; i < n * Pp; ++i) g[i] += 1.0f * dg[i]; /* add_scaled, optim.hpp:75-85 */
    free(gf);
    free(dg);
  }
  free(e);
  free(ge);
  free(x);
  cache_free(&c);
  return rc;
}

/* td3_update_step, algos.hpp:351-422: independent or shared-critic mode, optional
 * policy_member_mask and DvD policy-gradient hook */
int ora_td3_step_hook(ora_td3* st, const float* s, const float* a, const float* r,
                      const float* s2, const float* d, uint64_t b, const double* hyper,
                      const char* policy_mask, double* losses, const ora_dvd* dvd) {
  const uint64_t n = st->n, ds = st->ds, da = st->da, nc = st->nc;
  const int shared = st->shared;
  const uint64_t rc = shared ? n * b : b; /* critic rows per critic member (folded batch) */
  if (td3_validate(hyper, n)) return -2;
  float* y = (float*)malloc(sizeof(float) * n * b);
  ora_td3_target(st, s2, r, d, b, hyper, y);

  float* sa = concat(s, a, n, b, ds, da);
  const uint64_t Pc = st->cri.P, Pp = st->pol.P;
  float* g = (float*)malloc(sizeof(float) * n * (Pc > Pp ? Pc : Pp));
  if (losses) memset(losses, 0, sizeof(double) * 3 * n);
  for (int c = 0; c < 2; ++c) {
    float* params = st->net[2 + c];
    /* shared: critic_lr = {critic_lr[0]} (algos.hpp:366-367), one loss over n*b rows */
    mse_grads(&st->cri, params, nc, rc, sa, y, g, losses ? losses + c * n : NULL);
    for (uint64_t m = 0; m < nc; ++m) {
      adam_member(params + m * Pc, g + m * Pc, st->am[1 + c] + m * Pc, st->av[1 + c] + m * Pc,
                  &st->at[1 + c][m], Pc, HY(hyper, TH_CLR, n, m));
    }
  }

  char* fire = (char*)calloc(n, 1);
  int any = 0;
  for (uint64_t m = 0; m < n; ++m) {
    if (shared) {
      fire[m] = 1; /* one critic update per policy-population update (algos.hpp:382-384) */
    } else {
      st->delay_acc[m] += HY(hyper, TH_DELAY, n, m);
      if (st->delay_acc[m] >= 1.0 - 1e-12) {
        st->delay_acc[m] -= 1.0;
        fire[m] = 1;
      }
    }
    if (policy_mask && !policy_mask[m]) fire[m] = 0;
    any = any || fire[m];
  }
  int rc_hook = 0;

  if (any) {
    /* td3_policy_loss_grads, algos.hpp:318-338 */
    ora_cache cp, cq;
    mlp_forward(&st->pol, st->net[0], n, b, s, &cp);
    float* spa = concat(s, cp.out, n, b, ds, da);
    mlp_forward(&st->cri, st->net[2], nc, rc, spa, &cq);
    if (losses) {
      for (uint64_t m = 0; m < n; ++m) {
        double acc = 0.0;
        for (uint64_t i = 0; i < b; ++i) acc -= (double)cq.out[m * b + i];
        losses[2 * n + m] = fire[m] ? acc / (double)b : 0.0;
      }
    }
    float* gq = (float*)malloc(sizeof(float) * n * b);
    const float gval = -1.0f / (float)b;
    for (uint64_t i = 0; i < n * b; ++i) gq[i] = gval;
    float* gsa = (float*)malloc(sizeof(float) * n * b * (ds + da));
    mlp_backward(&st->cri, st->net[2], &cq, gq, g, gsa);
    float* ga = take_cols(gsa, n * b, ds + da, ds, da);
    mlp_backward(&st->pol, st->net[0], &cp, ga, g, NULL);
    if (dvd) rc_hook = dvd_hook(st, dvd, g);
    if (rc_hook == 0) {
      for (uint64_t m = 0; m < n; ++m) {
        if (!fire[m]) continue;
        adam_member(st->net[0] + m * Pp, g + m * Pp, st->am[0] + m * Pp, st->av[0] + m * Pp,
                    &st->at[0][m], Pp, HY(hyper, TH_PLR, n, m));
      }
      for (uint64_t m = 0; m < n; ++m) {
        if (!fire[m]) continue;
        polyak_member(st->net[1] + m * Pp, st->net[0] + m * Pp, Pp, HY(hyper, TH_TAU, n, m));
      }
      /* critic targets: per fired member, or the one shared critic with tau[0] (:407-418) */
      for (uint64_t m = 0; m < nc; ++m) {
        if (!shared && !fire[m]) continue;
        const double tau = HY(hyper, TH_TAU, n, m);
        polyak_member(st->net[4] + m * Pc, st->net[2] + m * Pc, Pc, tau);
        polyak_member(st->net[5] + m * Pc, st->net[3] + m * Pc, Pc, tau);
      }
    }
    free(spa);
    free(gq);
    free(gsa);
    free(ga);
    cache_free(&cp);
    cache_free(&cq);
  }
  if (rc_hook == 0) {
    for (uint64_t m = 0; m < n; ++m) st->steps[m] += 1;
  }
  free(fire);
  free(g);
  free(sa);
  free(y);
  return rc_hook;
}

int ora_td3_step(ora_td3* st, const float* s, const float* a, const float* r, const float* s2,
                 const float* d, uint64_t b, const double* hyper, const char* policy_mask,
                 double* losses) {
  return ora_td3_step_hook(st, s, a, r, s2, d, b, hyper, policy_mask, losses, NULL);
}

/* ------------------------------------------------------------------ CEM (evolve.hpp:221-297) */
void ora_cem_sample(const double* mean, const double* var, double noise, uint64_t dim,
                    uint64_t count, uint64_t key, uint64_t* next, double* out) {
  for (uint64_t c = 0; c < count; ++c) {
    for (uint64_t i = 0; i < dim; ++i) {
      const uint64_t ctr = *next;
      *next += 2;
      out[c * dim + i] = mean[i] + sqrt(var[i] + noise) * ora_normal_pair(key, ctr);
    }
  }
}

static const double* g_cem_scores;
static int cem_cmp(const void* pa, const void* pb) {
  const uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
  if (g_cem_scores[a] > g_cem_scores[b]) return -1;
  if (g_cem_scores[b] > g_cem_scores[a]) return 1;
  return a < b ? -1 : (a > b ? 1 : 0); /* stable_sort: ties keep index order */
}

int ora_cem_update(double* mean, double* var, double* noise, double noise_final,
                   double noise_decay, double elite_fraction, uint64_t dim, const double* cands,
                   const double* scores, uint64_t count) {
  if (count < 2 || count % 2 != 0) return -2;
  for (uint64_t i = 0; i < count; ++i) {
    if (!isfinite(scores[i])) return -2;
  }
  uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * count);
  for (uint64_t i = 0; i < count; ++i) order[i] = i;
  g_cem_scores = scores;
  qsort(order, count, sizeof(uint64_t), cem_cmp);
  const uint64_t elite = (uint64_t)(elite_fraction * (double)count);
  for (uint64_t i = 0; i < dim; ++i) mean[i] = 0.0;
  for (uint64_t e = 0; e < elite; ++e) {
    const double* c = cands + order[e] * dim;
    for (uint64_t i = 0; i < dim; ++i) mean[i] += c[i];
  }
  for (uint64_t i = 0; i < dim; ++i) mean[i] /= (double)elite;
  for (uint64_t i = 0; i < dim; ++i) var[i] = 0.0;
  for (uint64_t e = 0; e < elite; ++e) {
    const double* c = cands + order[e] * dim;
    for (uint64_t i = 0; i < dim; ++i) {
      const double dd = c[i] - mean[i];
      var[i] += dd * dd;
    }
  }
  for (uint64_t i = 0; i < dim; ++i) var[i] /= (double)elite;
  const double nn = *noise * noise_decay;
  *noise = noise_final < nn ? nn : noise_final; /* std::max(noise_final, noise * decay) */
  free(order);
  return 0;
}

/* ------------------------------------------------------------------ SAC (algos.hpp:470-837) */
struct ora_sac {
  uint64_t n, ds, da;
  uint64_t nc;  /* critic population: n, or 1 in shared-critic mode (algos.hpp:506) */
  int shared;
  ora_net pol, cri;
  float bound;
  uint64_t seed;
  float* net[6]; /* index 1 unused */
  float* am[3];
  float* av[3];
  int64_t* at[3];
  float* log_alpha;
  float* alpha_m;
  float* alpha_v;
  int64_t* alpha_t;
  uint64_t* steps;
  uint64_t* streams;
};

static const ora_net* sac_shape(const ora_sac* st, int net) {
  return net == 0 ? &st->pol : &st->cri;
}

ora_sac* ora_sac_create_mode(uint64_t n, uint64_t ds, uint64_t da, const uint64_t* hidden,
                             uint32_t nh, double bound, uint64_t seed, int shared) {
  ora_sac* st = (ora_sac*)calloc(1, sizeof(ora_sac));
  st->n = n;
  st->shared = shared ? 1 : 0;
  st->nc = shared ? 1 : n;
  const uint64_t nc = st->nc;
  st->ds = ds;
  st->da = da;
  st->bound = (float)bound;
  st->seed = seed;
  uint64_t dims[ORA_MAXL + 1];
  dims[0] = ds;
  for (uint32_t i = 0; i < nh; ++i) dims[i + 1] = hidden[i];
  dims[nh + 1] = 2 * da;
  net_make(&st->pol, dims, (int)nh + 2, ACT_NONE, 1.0f);
  dims[0] = ds + da;
  dims[nh + 1] = 1;
  net_make(&st->cri, dims, (int)nh + 2, ACT_NONE, 1.0f);
  for (int k = 0; k < 6; ++k) {
    if (k == 1) continue;
    st->net[k] = (float*)calloc((k == 0 ? n : nc) * sac_shape(st, k)->P, sizeof(float));
  }
  net_init(&st->pol, st->net[0], n, ora_mix64(seed ^ 0xD4));
  net_init(&st->cri, st->net[2], nc, ora_mix64(seed ^ 0xE5));
  net_init(&st->cri, st->net[3], nc, ora_mix64(seed ^ 0xF6));
  memcpy(st->net[4], st->net[2], sizeof(float) * nc * st->cri.P);
  memcpy(st->net[5], st->net[3], sizeof(float) * nc * st->cri.P);
  for (int k = 0; k < 3; ++k) {
    const uint64_t P = (k == 0) ? st->pol.P : st->cri.P;
    const uint64_t cnt = (k == 0) ? n : nc;
    st->am[k] = (float*)calloc(cnt * P, sizeof(float));
    st->av[k] = (float*)calloc(cnt * P, sizeof(float));
    st->at[k] = (int64_t*)calloc(cnt, sizeof(int64_t));
  }
  st->log_alpha = (float*)calloc(n, sizeof(float));
  st->alpha_m = (float*)calloc(n, sizeof(float));
  st->alpha_v = (float*)calloc(n, sizeof(float));
  st->alpha_t = (int64_t*)calloc(n, sizeof(int64_t));
  st->steps = (uint64_t*)calloc(n, sizeof(uint64_t));
  st->streams = (uint64_t*)calloc(n, sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) st->streams[i] = i;
  return st;
}

ora_sac* ora_sac_create(uint64_t n, uint64_t ds, uint64_t da, const uint64_t* hidden,
                        uint32_t nh, double bound, uint64_t seed) {
  return ora_sac_create_mode(n, ds, da, hidden, nh, bound, seed, 0);
}

void ora_sac_destroy(ora_sac* st) {
  if (!st) return;
  for (int k = 0; k < 6; ++k) free(st->net[k]);
  for (int k = 0; k < 3; ++k) {
    free(st->am[k]);
    free(st->av[k]);
    free(st->at[k]);
  }
  free(st->log_alpha);
  free(st->alpha_m);
  free(st->alpha_v);
  free(st->alpha_t);
  free(st->steps);
  free(st->streams);
  free(st);
}

uint64_t ora_sac_param_count(const ora_sac* st, int net) { return sac_shape(st, net)->P; }

void ora_sac_get_net(const ora_sac* st, int net, uint64_t m, float* out) {
  const uint64_t P = sac_shape(st, net)->P;
  memcpy(out, st->net[net] + m * P, sizeof(float) * P);
}

void ora_sac_set_net(ora_sac* st, int net, uint64_t m, const float* in) {
  const uint64_t P = sac_shape(st, net)->P;
  memcpy(st->net[net] + m * P, in, sizeof(float) * P);
}

void ora_sac_get_adam(const ora_sac* st, int net, uint64_t m, float* mo, float* vo, int64_t* t) {
  const int k = td3_opt_index(net);
  const uint64_t P = sac_shape(st, net)->P;
  memcpy(mo, st->am[k] + m * P, sizeof(float) * P);
  memcpy(vo, st->av[k] + m * P, sizeof(float) * P);
  *t = st->at[k][m];
}

void ora_sac_get_alpha(const ora_sac* st, float* log_alpha, float* am, float* av, int64_t* at,
                       uint64_t* steps) {
  memcpy(log_alpha, st->log_alpha, sizeof(float) * st->n);
  memcpy(am, st->alpha_m, sizeof(float) * st->n);
  memcpy(av, st->alpha_v, sizeof(float) * st->n);
  memcpy(at, st->alpha_t, sizeof(int64_t) * st->n);
  memcpy(steps, st->steps, sizeof(uint64_t) * st->n);
}

enum { SH_PLR = 0, SH_CLR, SH_ALR, SH_TE, SH_RS, SH_GAMMA, SH_TAU };

/* log_one_minus_tanh_sq, algos.hpp:523-529 */
static float l1mts(float x) {
  const float z = -2.0f * x;
  const float sp = maxf_(z, 0.0f) + log1pf(expf(-fabsf(z)));
  return (float)1.3862943611198906 - 2.0f * x - 2.0f * sp;
}

/* split_policy_head, algos.hpp:599-616: mu, clamped log_std, clamp flags; all [cnt][da] */
static void split_head(const float* h, uint64_t cnt, uint64_t da, float* mu, float* ls,
                       char* clamped) {
  for (uint64_t i = 0; i < cnt; ++i) {
    for (uint64_t j = 0; j < da; ++j) {
      mu[i * da + j] = h[i * 2 * da + j];
      float v = h[i * 2 * da + da + j];
      char c = 0;
      if (v < (float)-20.0) {
        v = (float)-20.0;
        c = 1;
      } else if (v > (float)2.0) {
        v = (float)2.0;
        c = 1;
      }
      ls[i * da + j] = v;
      clamped[i * da + j] = c;
    }
  }
}

/* act, algos.hpp:895-915: tanh policy output (already scaled by the bound) plus clipped
 * Gaussian exploration noise; std per member in action-bound units, stream (seed, streams[m],
 * kExploreNoise, steps[m]), counter 2e over the member's [rows][da] block.  out [n][rows][da]. */
void ora_td3_act(const ora_td3* st, const float* obs, uint64_t rows, const double* noise_std,
                 uint64_t seed, const uint64_t* steps, int deterministic, float* out) {
  ora_cache c;
  mlp_forward(&st->pol, st->net[0], st->n, rows, obs, &c);
  const uint64_t per = rows * st->da;
  memcpy(out, c.out, sizeof(float) * st->n * per);
  cache_free(&c);
  if (deterministic) return;
  const float bound = st->pol.out_scale;
  for (uint64_t m = 0; m < st->n; ++m) {
    if (noise_std[m] == 0.0) continue;
    const uint64_t key = ora_stream_key(seed, st->streams[m], USE_EXPLORE, steps[m]);
    const float sd = (float)(noise_std[m] * (double)bound);
    float* am = out + m * per;
    for (uint64_t e = 0; e < per; ++e)
      am[e] = clampf_(am[e] + (float)ora_normal_pair(key, 2 * e) * sd, -bound, bound);
  }
}

/* sac_act, algos.hpp:918-942: a = bound * tanh(mu + exp(log_std) * eps) (the mode when
 * deterministic), log_std clamped by split_policy_head. */
void ora_sac_act(const ora_sac* st, const float* obs, uint64_t rows, uint64_t seed,
                 const uint64_t* steps, int deterministic, float* out) {
  ora_cache c;
  mlp_forward(&st->pol, st->net[0], st->n, rows, obs, &c);
  const uint64_t cnt = st->n * rows, da = st->da, per = rows * da;
  float* mu = (float*)malloc(sizeof(float) * cnt * da);
  float* ls = (float*)malloc(sizeof(float) * cnt * da);
  char* cl = (char*)malloc(cnt * da);
  split_head(c.out, cnt, da, mu, ls, cl);
  cache_free(&c);
  if (!deterministic) {
    for (uint64_t m = 0; m < st->n; ++m) {
      const uint64_t key = ora_stream_key(seed, st->streams[m], USE_EXPLORE, steps[m]);
      for (uint64_t e = 0; e < per; ++e)
        mu[m * per + e] += expf(ls[m * per + e]) * (float)ora_normal_pair(key, 2 * e);
    }
  }
  for (uint64_t i = 0; i < cnt * da; ++i) out[i] = tanhf(mu[i]) * st->bound;
  free(mu);
  free(ls);
  free(cl);
}

/* draw_eps, algos.hpp:618-629 */
static void draw_eps(const ora_sac* st, uint64_t b, uint64_t use, float* eps) {
  const uint64_t da = st->da;
  for (uint64_t m = 0; m < st->n; ++m) {
    const uint64_t key = ora_stream_key(st->seed, st->streams[m], use, st->steps[m]);
    for (uint64_t e = 0; e < b * da; ++e) eps[m * b * da + e] = (float)ora_normal_pair(key, 2 * e);
  }
}

/* tanh_gaussian_logprob, algos.hpp:534-566; logp [n*b], x [n*b*da] */
static void tg_logprob(const float* mu, const float* ls, const float* eps, uint64_t nb,
                       uint64_t da, float bound, float* logp, float* x) {
  const float hl2pi = (float)0.9189385332046727;
  const float lb = logf(bound);
  for (uint64_t i = 0; i < nb; ++i) {
    float acc = 0.0f;
    for (uint64_t j = 0; j < da; ++j) {
      const uint64_t k = i * da + j;
      const float sig = expf(ls[k]);
      const float xv = mu[k] + sig * eps[k];
      x[k] = xv;
      acc += -0.5f * eps[k] * eps[k] - ls[k] - hl2pi;
      acc -= l1mts(xv);
      acc -= lb;
    }
    logp[i] = acc;
  }
}

/* sac_critic_target, algos.hpp:739-776 */
static void sac_target(const ora_sac* st, const float* s2, const float* r, const float* d,
                       uint64_t b, const double* hyper, float* y) {
  const uint64_t n = st->n, ds = st->ds, da = st->da, nb = n * b;
  ora_cache cp;
  mlp_forward(&st->pol, st->net[0], n, b, s2, &cp);
  float* mu = (float*)malloc(sizeof(float) * nb * da);
  float* ls = (float*)malloc(sizeof(float) * nb * da);
  char* cl = (char*)malloc(nb * da);
  float* eps = (float*)malloc(sizeof(float) * nb * da);
  float* x = (float*)malloc(sizeof(float) * nb * da);
  float* lp = (float*)malloc(sizeof(float) * nb);
  split_head(cp.out, nb, da, mu, ls, cl);
  draw_eps(st, b, USE_SAC_EPS_T, eps);
  tg_logprob(mu, ls, eps, nb, da, st->bound, lp, x);
  for (uint64_t k = 0; k < nb * da; ++k) x[k] = tanhf(x[k]);
  for (uint64_t k = 0; k < nb * da; ++k) x[k] *= st->bound;
  float* sa2 = concat(s2, x, n, b, ds, da);
  ora_cache c1, c2;
  const uint64_t rc = st->shared ? nb : b; /* critic_forward folding (algos.hpp:219-227) */
  mlp_forward(&st->cri, st->net[4], st->nc, rc, sa2, &c1);
  mlp_forward(&st->cri, st->net[5], st->nc, rc, sa2, &c2);
  for (uint64_t m = 0; m < n; ++m) {
    const float g = (float)HY(hyper, SH_GAMMA, n, m);
    const float rs = (float)HY(hyper, SH_RS, n, m);
    const float alpha = expf(st->log_alpha[m]);
    for (uint64_t i = 0; i < b; ++i) {
      const uint64_t k = m * b + i;
      const float qmin = minf_(c1.out[k], c2.out[k]);
      y[k] = rs * r[k] + g * (1.0f - d[k]) * (qmin - alpha * lp[k]);
    }
  }
  free(mu);
  free(ls);
  free(cl);
  free(eps);
  free(x);
  free(lp);
  free(sa2);
  cache_free(&cp);
  cache_free(&c1);
  cache_free(&c2);
}

/* sac_update_step, algos.hpp:781-837, with sac_policy_loss_grads (:643-735) inlined */
int ora_sac_step(ora_sac* st, const float* s, const float* a, const float* r, const float* s2,
                 const float* d, uint64_t b, const double* hyper, double* losses) {
  const uint64_t n = st->n, ds = st->ds, da = st->da, nb = n * b;
  const uint64_t Pc = st->cri.P, Pp = st->pol.P;
  double* alpha = (double*)malloc(sizeof(double) * n);
  for (uint64_t m = 0; m < n; ++m) alpha[m] = exp((double)st->log_alpha[m]);

  float* y = (float*)malloc(sizeof(float) * nb);
  sac_target(st, s2, r, d, b, hyper, y);
  float* sa = concat(s, a, n, b, ds, da);
  float* g = (float*)malloc(sizeof(float) * n * (Pc > Pp ? Pc : Pp));
  const uint64_t nc = st->nc, rc = st->shared ? nb : b;
  if (losses) memset(losses, 0, sizeof(double) * 3 * n);
  for (int c = 0; c < 2; ++c) {
    float* params = st->net[2 + c];
    mse_grads(&st->cri, params, nc, rc, sa, y, g, losses ? losses + c * n : NULL);
    for (uint64_t m = 0; m < nc; ++m) {
      adam_member(params + m * Pc, g + m * Pc, st->am[1 + c] + m * Pc, st->av[1 + c] + m * Pc,
                  &st->at[1 + c][m], Pc, HY(hyper, SH_CLR, n, m));
    }
  }

  /* policy loss and gradients */
  float* eps = (float*)malloc(sizeof(float) * nb * da);
  draw_eps(st, b, USE_SAC_EPS, eps);
  ora_cache cp;
  mlp_forward(&st->pol, st->net[0], n, b, s, &cp);
  float* mu = (float*)malloc(sizeof(float) * nb * da);
  float* ls = (float*)malloc(sizeof(float) * nb * da);
  char* cl = (char*)malloc(nb * da);
  float* x = (float*)malloc(sizeof(float) * nb * da);
  float* lp = (float*)malloc(sizeof(float) * nb);
  split_head(cp.out, nb, da, mu, ls, cl);
  tg_logprob(mu, ls, eps, nb, da, st->bound, lp, x);
  float* th = (float*)malloc(sizeof(float) * nb * da);
  float* act = (float*)malloc(sizeof(float) * nb * da);
  for (uint64_t k = 0; k < nb * da; ++k) {
    th[k] = tanhf(x[k]);
    act[k] = th[k] * st->bound;
  }
  float* spa = concat(s, act, n, b, ds, da);
  ora_cache c1, c2;
  mlp_forward(&st->cri, st->net[2], nc, rc, spa, &c1);
  mlp_forward(&st->cri, st->net[3], nc, rc, spa, &c2);
  float* gq1 = (float*)calloc(nb, sizeof(float));
  float* gq2 = (float*)calloc(nb, sizeof(float));
  float* lw = (float*)malloc(sizeof(float) * nb);
  const float inv_rows = 1.0f / (float)b;
  for (uint64_t m = 0; m < n; ++m) {
    const float am = (float)alpha[m];
    double lsum = 0.0;
    for (uint64_t i = 0; i < b; ++i) {
      const uint64_t k = m * b + i;
      const float qmin = minf_(c1.out[k], c2.out[k]);
      lsum += (double)(am * lp[k] - qmin) / (double)b;
      lw[k] = am * inv_rows;
      if (c1.out[k] <= c2.out[k]) gq1[k] = -inv_rows;
      else gq2[k] = -inv_rows;
    }
    if (losses) losses[2 * n + m] = lsum;
  }
  float* gsa1 = (float*)malloc(sizeof(float) * nb * (ds + da));
  float* gsa2 = (float*)malloc(sizeof(float) * nb * (ds + da));
  mlp_backward(&st->cri, st->net[2], &c1, gq1, g, gsa1);
  mlp_backward(&st->cri, st->net[3], &c2, gq2, g, gsa2);
  for (uint64_t i = 0; i < nb * (ds + da); ++i) gsa1[i] += gsa2[i];
  float* ga = take_cols(gsa1, nb, ds + da, ds, da);
  /* tanh_gaussian_logprob_backward, algos.hpp:571-595, then the action path (:708-724) */
  float* gh = (float*)malloc(sizeof(float) * nb * 2 * da);
  for (uint64_t i = 0; i < nb; ++i) {
    const float w = lw[i];
    for (uint64_t j = 0; j < da; ++j) {
      const uint64_t k = i * da + j;
      const float dlogp_dx = 2.0f * tanhf(x[k]);
      float gmu = w * dlogp_dx;
      float gls = w * (dlogp_dx * expf(ls[k]) * eps[k] - 1.0f);
      const float dadx = st->bound * (1.0f - th[k] * th[k]);
      const float gx = ga[k] * dadx;
      gmu += gx;
      gls += gx * expf(ls[k]) * eps[k];
      if (cl[k]) gls = 0.0f;
      gh[i * 2 * da + j] = gmu;
      gh[i * 2 * da + da + j] = gls;
    }
  }
  mlp_backward(&st->pol, st->net[0], &cp, gh, g, NULL);
  for (uint64_t m = 0; m < n; ++m) {
    adam_member(st->net[0] + m * Pp, g + m * Pp, st->am[0] + m * Pp, st->av[0] + m * Pp,
                &st->at[0][m], Pp, HY(hyper, SH_PLR, n, m));
  }
  /* temperature, algos.hpp:814-825 */
  for (uint64_t m = 0; m < n; ++m) {
    double mt = 0.0;
    for (uint64_t i = 0; i < b; ++i) mt += (double)lp[m * b + i] + HY(hyper, SH_TE, n, m);
    mt /= (double)b;
    const float ga1 = (float)(-alpha[m] * mt);
    adam_member(&st->log_alpha[m], &ga1, &st->alpha_m[m], &st->alpha_v[m], &st->alpha_t[m], 1,
                HY(hyper, SH_ALR, n, m));
  }
  for (uint64_t m = 0; m < nc; ++m) { /* shared: {tau[0]} on the one critic (:827-834) */
    const double tau = HY(hyper, SH_TAU, n, m);
    polyak_member(st->net[4] + m * Pc, st->net[2] + m * Pc, Pc, tau);
    polyak_member(st->net[5] + m * Pc, st->net[3] + m * Pc, Pc, tau);
  }
  for (uint64_t m = 0; m < n; ++m) st->steps[m] += 1;

  free(alpha);
  free(y);
  free(sa);
  free(g);
  free(eps);
  free(mu);
  free(ls);
  free(cl);
  free(x);
  free(lp);
  free(th);
  free(act);
  free(spa);
  free(gq1);
  free(gq2);
  free(lw);
  free(gsa1);
  free(gsa2);
  free(ga);
  free(gh);
  cache_free(&cp);
  cache_free(&c1);
  cache_free(&c2);
  return 0;
}

/* ------------------------------------------------------------------ synthetic batches */
void ora_synthetic_batches(uint64_t count, uint64_t n, uint64_t b, uint64_t ds, uint64_t da,
                           uint64_t seed, float* s, float* a, float* r, float* s2, float* d) {
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t ks = ora_stream_key(seed, i, USE_GENERIC, 1);
    const uint64_t ka = ora_stream_key(seed, i, USE_GENERIC, 2);
    const uint64_t kr = ora_stream_key(seed, i, USE_GENERIC, 3);
    const uint64_t k2 = ora_stream_key(seed, i, USE_GENERIC, 4);
    const uint64_t kd = ora_stream_key(seed, i, USE_GENERIC, 5);
    for (uint64_t e = 0; e < n * b * ds; ++e) s[i * n * b * ds + e] = (float)uniform_in(ks, e, -1.0, 1.0);
    for (uint64_t e = 0; e < n * b * da; ++e) a[i * n * b * da + e] = (float)uniform_in(ka, e, -1.0, 1.0);
    for (uint64_t e = 0; e < n * b; ++e) r[i * n * b + e] = (float)uniform_in(kr, e, -1.0, 1.0);
    for (uint64_t e = 0; e < n * b * ds; ++e) s2[i * n * b * ds + e] = (float)uniform_in(k2, e, -1.0, 1.0);
    for (uint64_t e = 0; e < n * b; ++e) d[i * n * b + e] = ora_uniform(kd, e) < 0.02 ? 1.0f : 0.0f;
  }
}

/* ------------------------------------------------------------------ replay (replay.hpp) */
struct ora_replay {
  uint64_t cap, ds, da, inserts;
  float *s, *a, *s2, *r, *d;
  uint32_t* member;
};

ora_replay* ora_replay_create(uint64_t cap, uint64_t ds, uint64_t da) {
  ora_replay* rb = (ora_replay*)calloc(1, sizeof(ora_replay));
  rb->cap = cap;
  rb->ds = ds;
  rb->da = da;
  rb->s = (float*)calloc(cap * ds, sizeof(float));
  rb->a = (float*)calloc(cap * da, sizeof(float));
  rb->s2 = (float*)calloc(cap * ds, sizeof(float));
  rb->r = (float*)calloc(cap, sizeof(float));
  rb->d = (float*)calloc(cap, sizeof(float));
  rb->member = (uint32_t*)calloc(cap, sizeof(uint32_t));
  return rb;
}

void ora_replay_destroy(ora_replay* rb) {
  if (!rb) return;
  free(rb->s);
  free(rb->a);
  free(rb->s2);
  free(rb->r);
  free(rb->d);
  free(rb->member);
  free(rb);
}

/* ReplayBuffer::push, replay.hpp:56-69 */
void ora_replay_push(ora_replay* rb, const float* s, const float* a, float r, const float* s2,
                     float d, uint32_t member) {
  const uint64_t slot = rb->inserts % rb->cap;
  memcpy(rb->s + slot * rb->ds, s, sizeof(float) * rb->ds);
  memcpy(rb->a + slot * rb->da, a, sizeof(float) * rb->da);
  memcpy(rb->s2 + slot * rb->ds, s2, sizeof(float) * rb->ds);
  rb->r[slot] = r;
  rb->d[slot] = d;
  rb->member[slot] = member;
  rb->inserts++;
}

uint64_t ora_replay_size(const ora_replay* rb) {
  return rb->inserts < rb->cap ? rb->inserts : rb->cap;
}

/* sample_batch + fill_member_rows, replay.hpp:181-204 and :91-111 */
int ora_sample_batch(ora_replay** bufs, uint64_t nbufs, uint64_t b, int mode, uint64_t members,
                     uint64_t seed, const uint64_t* streams, uint64_t draw_id, uint64_t min_size,
                     float* s, float* a, float* r, float* s2, float* d, uint64_t* slots) {
  if (nbufs == 0 || (mode == 0 && nbufs != members)) return -2;
  for (uint64_t m = 0; m < members; ++m) {
    const ora_replay* src = (mode == 0) ? bufs[m] : bufs[0];
    const uint64_t key = ora_stream_key(seed, streams[m], USE_SAMPLE, draw_id);
    const uint64_t size = ora_replay_size(src);
    const uint64_t need = min_size > 1 ? min_size : 1;
    if (size < need) return 0;
    const uint64_t ds = src->ds, da = src->da;
    for (uint64_t i = 0; i < b; ++i) {
      const uint64_t slot = ora_bits(key, i) % size;
      if (slots) slots[m * b + i] = slot;
      memcpy(s + (m * b + i) * ds, src->s + slot * ds, sizeof(float) * ds);
      memcpy(a + (m * b + i) * da, src->a + slot * da, sizeof(float) * da);
      memcpy(s2 + (m * b + i) * ds, src->s2 + slot * ds, sizeof(float) * ds);
      r[m * b + i] = src->r[slot];
      d[m * b + i] = src->d[slot];
    }
  }
  return 1;
}

/* ------------------------------------------------------------------ PBT (evolve.hpp) */
static double mean_return(const double* rings, const uint32_t* counts, uint64_t ring_cap,
                          uint64_t m) {
  double acc = 0.0;
  for (uint32_t j = 0; j < counts[m]; ++j) acc += rings[m * ring_cap + j];
  return acc / (double)counts[m];
}

/* pbt_rank, evolve.hpp:112-122: stable sort, best first, ties toward the lower index */
int ora_pbt_rank(const double* rings, const uint32_t* counts, uint64_t n, uint64_t ring_cap,
                 uint64_t* order) {
  if (n == 0) return -4;
  for (uint64_t m = 0; m < n; ++m) {
    if (counts[m] == 0) return -4;
  }
  double* mean = (double*)malloc(sizeof(double) * n);
  for (uint64_t m = 0; m < n; ++m) mean[m] = mean_return(rings, counts, ring_cap, m);
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t key = i;
    uint64_t j = i;
    while (j > 0 && mean[key] > mean[order[j - 1]]) {
      order[j] = order[j - 1];
      --j;
    }
    order[j] = key;
  }
  free(mean);
  return 0;
}

/* pbt_plan, evolve.hpp:133-145 */
int ora_pbt_plan(const double* rings, const uint32_t* counts, uint64_t n, uint64_t ring_cap,
                 double trunc, uint64_t rng_key, uint64_t* rng_next, uint64_t* replaced,
                 uint64_t* donors) {
  if (n < 4) return 0;
  uint64_t* order = (uint64_t*)malloc(sizeof(uint64_t) * n);
  const int rc = ora_pbt_rank(rings, counts, n, ring_cap, order);
  if (rc) {
    free(order);
    return rc;
  }
  const uint64_t cut = (uint64_t)ceil(trunc * (double)n);
  for (uint64_t i = 0; i < cut; ++i) {
    replaced[i] = order[n - 1 - i];
    donors[i] = order[seq_bits(rng_key, rng_next) % cut];
  }
  free(order);
  return (int)cut;
}

/* Td3Prior::sample_member, evolve.hpp:31-49 (untuned fields reset to Td3Hyper::defaults) */
void ora_td3_prior_sample(uint64_t key, uint64_t* next, double* h) {
  h[TH_CLR] = seq_log_uniform(key, next, 3e-5, 3e-3);
  h[TH_PLR] = seq_log_uniform(key, next, 3e-5, 3e-3);
  h[TH_DELAY] = seq_uniform(key, next, 0.2, 1.0);
  h[TH_EXPLORE] = seq_uniform(key, next, 0.0, 1.0);
  h[TH_TSTD] = seq_uniform(key, next, 0.0, 1.0);
  h[TH_GAMMA] = seq_uniform(key, next, 0.9, 1.0);
  h[TH_TCLIP] = 0.5;
  h[TH_TAU] = 0.005;
}

/* SacPrior::sample_member, evolve.hpp:54-73 */
void ora_sac_prior_sample(uint64_t key, uint64_t* next, double default_te, double* h) {
  h[SH_PLR] = seq_log_uniform(key, next, 3e-5, 3e-3);
  h[SH_CLR] = seq_log_uniform(key, next, 3e-5, 3e-3);
  h[SH_ALR] = seq_log_uniform(key, next, 3e-5, 3e-3);
  h[SH_TE] = seq_uniform(key, next, 0.2, 2.0) * default_te;
  h[SH_RS] = seq_uniform(key, next, 0.1, 10.0);
  h[SH_GAMMA] = seq_uniform(key, next, 0.9, 1.0);
  h[SH_TAU] = 0.005;
}

/* pbt_evolve_trainer (TD3), evolve.hpp:169-190 */
int ora_td3_pbt_evolve(ora_td3* st, const double* rings, const uint32_t* counts,
                       uint64_t ring_cap, double* hyper, uint64_t rng_key, uint64_t* rng_next,
                       uint64_t* replaced, uint64_t* donors) {
  const uint64_t n = st->n;
  const int cnt = ora_pbt_plan(rings, counts, n, ring_cap, 0.3, rng_key, rng_next, replaced, donors);
  if (cnt <= 0) return cnt;
  if (st->shared) return -3; /* copy_member on the 1-member critic: UsageError (net_pop.hpp:194) */
  for (int i = 0; i < cnt; ++i) {
    const uint64_t dst = replaced[i], src = donors[i];
    for (int k = 0; k < 6; ++k) {
      const uint64_t P = td3_shape(st, k)->P;
      if (src != dst) memcpy(st->net[k] + dst * P, st->net[k] + src * P, sizeof(float) * P);
    }
    for (int k = 0; k < 3; ++k) {
      const uint64_t P = (k == 0) ? st->pol.P : st->cri.P;
      memset(st->am[k] + dst * P, 0, sizeof(float) * P);
      memset(st->av[k] + dst * P, 0, sizeof(float) * P);
      st->at[k][dst] = 0;
    }
    st->delay_acc[dst] = 0.0;
    double h[8];
    ora_td3_prior_sample(rng_key, rng_next, h);
    for (int f = 0; f < 8; ++f) HY(hyper, f, n, dst) = h[f];
  }
  return cnt;
}

/* pbt_evolve_trainer (SAC), evolve.hpp:192-213 */
int ora_sac_pbt_evolve(ora_sac* st, const double* rings, const uint32_t* counts,
                       uint64_t ring_cap, double* hyper, double default_te, uint64_t rng_key,
                       uint64_t* rng_next, uint64_t* replaced, uint64_t* donors) {
  const uint64_t n = st->n;
  const int cnt = ora_pbt_plan(rings, counts, n, ring_cap, 0.3, rng_key, rng_next, replaced, donors);
  if (cnt <= 0) return cnt;
  if (st->shared) return -3; /* copy_member on the 1-member critic: UsageError (net_pop.hpp:194) */
  for (int i = 0; i < cnt; ++i) {
    const uint64_t dst = replaced[i], src = donors[i];
    for (int k = 0; k < 6; ++k) {
      if (k == 1) continue;
      const uint64_t P = sac_shape(st, k)->P;
      if (src != dst) memcpy(st->net[k] + dst * P, st->net[k] + src * P, sizeof(float) * P);
    }
    st->log_alpha[dst] = st->log_alpha[src];
    for (int k = 0; k < 3; ++k) {
      const uint64_t P = (k == 0) ? st->pol.P : st->cri.P;
      memset(st->am[k] + dst * P, 0, sizeof(float) * P);
      memset(st->av[k] + dst * P, 0, sizeof(float) * P);
      st->at[k][dst] = 0;
    }
    st->alpha_m[dst] = 0.0f;
    st->alpha_v[dst] = 0.0f;
    st->alpha_t[dst] = 0;
    double h[7];
    ora_sac_prior_sample(rng_key, rng_next, default_te, h);
    for (int f = 0; f < 7; ++f) HY(hyper, f, n, dst) = h[f];
  }
  return cnt;
}
