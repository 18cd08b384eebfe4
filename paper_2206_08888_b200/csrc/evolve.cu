// Population-level search around the update step: the DvD diversity
// hook on the policy gradients (evolve.hpp:304-525) and CEM over flat policy vectors
// (evolve.hpp:221-297).
//
// DvD: dvd_policy_hook reads only the policies, which the update step does not touch before the
// hook runs (td3_update_step, algos.hpp:394-396: the critic step comes first), so the hook's
// whole computation runs as a pre-pass on the device before the step: the population forward on
// the probe states (the same fused forward kernels as the step), one D2H of the [n][M*da]
// embeddings, the n x n log-determinant loss on the host in double (the reference's own
// arithmetic: n is the population size, the kernel matrix is tiny), one H2D of d loss / d e, and
// the policy backward into a gradient arena that the step adds into the policy gradients right
// before the policy Adam.
//
// CEM: candidates are drawn on the device straight into the policy arena (one counter-based
// normal per coordinate, RngSequence counters next + 2 (c dim + i)), kept in double for the
// refit, which is a per-coordinate sum over the elites in score order (host stable sort of n
// scores).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "pop_impl.cuh"

namespace pbrl {

// ------------------------------------------------------------------ DvD host math
// dvd_loss (evolve.hpp:411-465), bit-for-bit the reference's double arithmetic
int dvd_loss_host(const double* emb, uint64_t n, uint64_t dim, double length_scale, double jitter,
                  double lambda, double* loss, double* logdet_out, double* grad) {
  if (n < 2) PBRL_THROW(PBRL_E_CONFIG, "dvd_loss: need at least two embedding rows");
  if (!(length_scale > 0)) PBRL_THROW(PBRL_E_CONFIG, "dvd_loss: length scale must be positive");
  // canonical_order (:391-405): stable lexicographic sort of the rows
  std::vector<uint64_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
    const double* ra = emb + a * dim;
    const double* rb = emb + b * dim;
    for (uint64_t k = 0; k < dim; ++k)
      if (ra[k] != rb[k]) return ra[k] < rb[k];
    return false;
  });
  const double inv2l2 = 1.0 / (2.0 * length_scale * length_scale);
  std::vector<double> kernel(n * n);
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
      const double kij = std::exp(-d2 * inv2l2);
      kernel[i * n + j] = kij;
      kernel[j * n + i] = kij;
    }
  }
  std::vector<double> m = kernel;
  for (uint64_t i = 0; i < n; ++i) m[i * n + i] += jitter;
  // cholesky (:352-367)
  for (uint64_t i = 0; i < n; ++i) {
    for (uint64_t j = 0; j <= i; ++j) {
      double sum = m[i * n + j];
      for (uint64_t k = 0; k < j; ++k) sum -= m[i * n + k] * m[j * n + k];
      if (i == j) {
        if (!(sum > 0.0))
          PBRL_THROW(PBRL_E_DEGENERATE,
                     "dvd_loss: kernel matrix is not positive definite even with jitter " +
                         std::to_string(jitter));
        m[i * n + i] = std::sqrt(sum);
      } else {
        m[i * n + j] = sum / m[j * n + j];
      }
    }
    for (uint64_t j = i + 1; j < n; ++j) m[i * n + j] = 0.0;
  }
  double logdet = 0;
  for (uint64_t i = 0; i < n; ++i) logdet += 2.0 * std::log(m[i * n + i]);
  // cholesky_inverse (:370-388)
  std::vector<double> minv(n * n), col(n);
  for (uint64_t c = 0; c < n; ++c) {
    for (uint64_t i = 0; i < n; ++i) {
      double sum = (i == c) ? 1.0 : 0.0;
      for (uint64_t k = 0; k < i; ++k) sum -= m[i * n + k] * col[k];
      col[i] = sum / m[i * n + i];
    }
    for (uint64_t ii = n; ii-- > 0;) {
      double sum = col[ii];
      for (uint64_t k = ii + 1; k < n; ++k) sum -= m[k * n + ii] * col[k];
      col[ii] = sum / m[ii * n + ii];
    }
    for (uint64_t i = 0; i < n; ++i) minv[i * n + c] = col[i];
  }
  if (logdet_out) *logdet_out = logdet;
  if (loss) *loss = -lambda * logdet;
  if (grad) {
    std::fill(grad, grad + n * dim, 0.0);
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
  return 0;
}

// median_pairwise_distance (evolve.hpp:469-486)
double median_pairwise_distance_host(const double* emb, uint64_t n, uint64_t dim) {
  std::vector<double> d;
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t j = i + 1; j < n; ++j) {
      double d2 = 0;
      for (uint64_t k = 0; k < dim; ++k) {
        const double x = emb[i * dim + k] - emb[j * dim + k];
        d2 += x * x;
      }
      d.push_back(std::sqrt(d2));
    }
  if (d.empty()) return 1.0;
  std::sort(d.begin(), d.end());
  const double med = d[d.size() / 2];
  return med > 0 ? med : 1.0;
}

// ------------------------------------------------------------------ DvD device kernels
// pre-activation cotangent of the tanh output layer: g = (grad * scale) * (1 - t^2), the order of
// pop_mlp_backward (net_pop.hpp:134-160 via activation_backward, pop_tensor.hpp:285-292)
__global__ void k_tanh_cotangent(long long rows, int da, int ld, const float* grad,
                                 const float* t, float scale, float* gz) {
  PDL_ENTRY();
  for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < rows * da;
       e += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = e / da;
    const int o = static_cast<int>(e - r * da);
    const float g = grad[e] * scale;
    const float tv = t[e];
    gz[r * ld + o] = g * (1.0f - tv * tv);
  }
}

// add_scaled(grads, dgrads, T(1)) (optim.hpp:75-85): acc += 1 * other
__global__ void k_add_into(float* acc, const float* other, size_t count) {
  PDL_ENTRY();
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    acc[i] += 1.0f * other[i];
}

void launch_add_into(float* acc, const float* other, size_t count, cudaStream_t s) {
  const int blocks = static_cast<int>(std::min<size_t>((count + 255) / 256, 148 * 8));
  launch_k(k_add_into, std::max(blocks, 1), 256, 0, s, acc, other, count);
}

__global__ void k_flag_convert(int* flag, float* flag_f, int to_float) {
  PDL_ENTRY();
  if (threadIdx.x == 0) {
    if (to_float) *flag_f = static_cast<float>(*flag);
    else *flag = *flag_f > 0.0f ? 1 : 0;
  }
}

void launch_flag_convert(int* flag, float* flag_f, int to_float, cudaStream_t s) {
  launch_k(k_flag_convert, 1, 32, 0, s, flag, flag_f, to_float);
}

void Pop::set_dvd(const double* probe, uint64_t m_states, double length_scale, double jitter,
                  double lambda) {
  if (!probe || lambda == 0.0) {  // dvd_policy_hook returns without effect at lambda 0
    if (dvd.on) invalidate_graphs();
    dvd.on = false;
    dvd.lambda = lambda;
    return;
  }
  if (algo != PBRL_ALGO_TD3) PBRL_THROW(PBRL_E_USAGE, "DvD policy hook: TD3 only (PolicyGradHook)");
  if (n_global != static_cast<uint64_t>(n))
    PBRL_THROW(PBRL_E_USAGE, "DvD policy hook: the kernel matrix spans the whole population "
                             "(single-shard populations only)");
  if (m_states < 1) PBRL_THROW(PBRL_E_SHAPE, "dvd_embed: probe matrix size != M * observation_dim");
  if (!(length_scale > 0)) PBRL_THROW(PBRL_E_CONFIG, "dvd_loss: length scale must be positive");
  if (n < 2) PBRL_THROW(PBRL_E_CONFIG, "dvd_loss: need at least two embedding rows");
  const int ms = static_cast<int>(m_states);
  if (!dvd.on) invalidate_graphs();  // the step graph gains the gradient add
  dvd.on = true;
  dvd.ls = length_scale;
  dvd.jitter = jitter;
  dvd.lambda = lambda;
  dvd.probe.assign(probe, probe + static_cast<size_t>(ms) * ds);
  const int L = pol.depth;
  const long long rows = static_cast<long long>(n) * ms;
  if (ms != dvd.ms) {
    dvd.ms = ms;
    dvd.ldx = padl(ds);
    dvd.x.alloc(rows * dvd.ldx);
    dvd.x.zero(stream);
    dvd.emb.alloc(rows * da);
    dvd.t.alloc(rows * da);
    dvd.gemb.alloc(rows * da);
    dvd.gz.alloc(rows * pad4(da));
    dvd.gz.zero(stream);
    dvd.h.clear();
    dvd.dh.clear();
    for (int l = 0; l + 1 < L; ++l) {
      const size_t h = static_cast<size_t>(padl(pol.dims[l + 1])) + (pol.dims[l + 1] + 31) / 32;
      for (auto* v : {&dvd.h, &dvd.dh}) {
        v->emplace_back();
        v->back().alloc(rows * h);
        v->back().zero(stream);
      }
    }
    dvd.obs.alloc(rows * ds);
  }
  dvd.grad.alloc(static_cast<size_t>(n) * pol.stride);
  // the probe block, replicated per member and cast to float (dvd_embed_cached, :319-335)
  std::vector<float> xs(static_cast<size_t>(rows) * ds);
  for (int m = 0; m < n; ++m)
    for (size_t i = 0; i < static_cast<size_t>(ms) * ds; ++i)
      xs[static_cast<size_t>(m) * ms * ds + i] = static_cast<float>(dvd.probe[i]);
  dvd.obs.upload(xs.data(), xs.size(), stream);
  launch_pack_obs(rows, ds, dvd.ldx, dvd.obs.p, dvd.x.p, act16() ? 1 : 0, stream);
  count_launch(1);
  sync();
}

// forward of the policies on the probe block: embeddings [n][M][da] (fp32) + tanh values
void Pop::dvd_forward() {
  const int ms = dvd.ms;
  const Mat x{dvd.x.p, static_cast<long long>(ms) * dvd.ldx, dvd.ldx, 0};
  mlp_forward(pol, pol_p.p, n, ms, x, dvd.h, dvd.emb.p, static_cast<long long>(ms) * da, da,
              EPI_BIAS_TANH, nullptr, dvd.t.p, static_cast<long long>(ms) * da, da, false, true,
              false);
}

void Pop::dvd_prepass() {
  if (!dvd.on) return;
  if (act16() && weights_dirty) refresh_shadows();
  const int ms = dvd.ms;
  const uint64_t dim = static_cast<uint64_t>(ms) * da;
  const size_t cnt = static_cast<size_t>(n) * dim;
  dvd_forward();
  std::vector<float> e(cnt);
  CUDA_CHECK(cudaMemcpyAsync(e.data(), dvd.emb.p, cnt * 4, cudaMemcpyDeviceToHost, stream));
  sync();
  std::vector<double> ed(e.begin(), e.end()), ge(cnt);
  dvd_loss_host(ed.data(), n, dim, dvd.ls, dvd.jitter, dvd.lambda, nullptr, nullptr, ge.data());
  for (size_t i = 0; i < cnt; ++i) e[i] = static_cast<float>(ge[i]);
  dvd.gemb.upload(e.data(), cnt, stream);
  const long long rows = static_cast<long long>(n) * ms;
  const int lt = pad4(da);
  timed(PC_ELEM, 0.0, 0.0, 0, [&] {
    const int blocks = static_cast<int>(std::min<long long>((rows * da + 255) / 256, 148 * 8));
    launch_k(k_tanh_cotangent, std::max(blocks, 1), 256, 0, stream, rows, da, lt, dvd.gemb.p,
             dvd.t.p, pol.out_scale, dvd.gz.p);
  });
  const Mat x0{dvd.x.p, static_cast<long long>(ms) * dvd.ldx, dvd.ldx, 0};
  mlp_backward(pol, pol_p.p, dvd.grad.p, n, ms, Mat{dvd.gz.p, static_cast<long long>(ms) * lt, lt, 0},
               x0, dvd.h, dvd.dh, nullptr, nullptr);
}

// ------------------------------------------------------------------ CEM
__global__ void k_cem_sample(const double* mean, const double* var, double noise, uint64_t dim,
                             uint64_t count, uint64_t key, uint64_t next0, double* cand,
                             float* arena, size_t stride) {
  PDL_ENTRY();
  const uint64_t total = dim * count;
  for (uint64_t e = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t c = e / dim, i = e - c * dim;
    // RngSequence::normal consumes counters (next, next+1) and advances by 2 (rng.hpp:88-92)
    const double v = mean[i] + sqrt(var[i] + noise) * rng_normal_pair(key, next0 + 2 * e);
    cand[e] = v;
    arena[c * stride + i] = static_cast<float>(v);  // unflatten_member of the T cast
  }
}

// elite refit (evolve.hpp:276-295): one thread per coordinate, elites in score order
__global__ void k_cem_refit(const double* cand, uint64_t dim, const uint64_t* order, int elite,
                            double* mean, double* var) {
  PDL_ENTRY();
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < dim;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    double m = 0.0;
    for (int e = 0; e < elite; ++e) m += cand[order[e] * dim + i];
    m /= static_cast<double>(elite);
    double v = 0.0;
    for (int e = 0; e < elite; ++e) {
      const double d = cand[order[e] * dim + i] - m;
      v += d * d;
    }
    mean[i] = m;
    var[i] = v / static_cast<double>(elite);
  }
}

Cem::Cem(Pop* p, const double* mean0, double init_var) : pop(p) {
  if (p->algo != PBRL_ALGO_TD3) PBRL_THROW(PBRL_E_USAGE, "CEM: TD3 policies only (pipeline_run.hpp:81)");
  if (p->n_global != static_cast<uint64_t>(p->n))
    PBRL_THROW(PBRL_E_USAGE, "CEM: the elite refit spans the whole population (single shard)");
  dim = p->pol.P;
  mean.alloc(dim);
  var.alloc(dim);
  cand.alloc(dim * static_cast<size_t>(p->n));
  cand.zero(p->stream);
  if (mean0) {
    mean.upload(mean0, dim, p->stream);
  } else {  // cem_init(flatten_member(policy, 0)) as run_training does (pipeline_run.hpp:159-162)
    std::vector<float> f(dim);
    CUDA_CHECK(cudaMemcpyAsync(f.data(), p->pol_p.p, dim * 4, cudaMemcpyDeviceToHost, p->stream));
    p->sync();
    std::vector<double> d(f.begin(), f.end());
    mean.upload(d.data(), dim, p->stream);
  }
  std::vector<double> v(dim, init_var);
  var.upload(v.data(), dim, p->stream);
  noise = noise_init;
  p->sync();
}

// cem_sample into the policy arena, then the rest of cem_resample (pipeline_run.hpp:148-158):
// targets = policies, policy Adam state reset
void Cem::resample(uint64_t key, uint64_t* next) {
  Pop* p = pop;
  const uint64_t count = static_cast<uint64_t>(p->n);
  const uint64_t total = dim * count;
  const int blocks = static_cast<int>(std::min<uint64_t>((total + 255) / 256, 148 * 16));
  launch_k(k_cem_sample, std::max(blocks, 1), 256, 0, p->stream, mean.p, var.p, noise, dim, count,
           key, *next, cand.p, p->pol_p.p, p->pol.stride);
  p->count_launch(1);
  *next += 2 * total;
  const size_t np = static_cast<size_t>(p->n) * p->pol.stride;
  CUDA_CHECK(cudaMemcpyAsync(p->pol_t.p, p->pol_p.p, np * 4, cudaMemcpyDeviceToDevice, p->stream));
  CUDA_CHECK(cudaMemsetAsync(p->pol_m.p, 0, np * 4, p->stream));
  CUDA_CHECK(cudaMemsetAsync(p->pol_v.p, 0, np * 4, p->stream));
  CUDA_CHECK(cudaMemsetAsync(p->t_pol.p, 0, 8 * p->n, p->stream));
  p->weights_dirty = true;
  p->weights_written_outside();
  sampled = true;
  p->sync();
}

void Cem::update(const double* scores, uint64_t count) {
  Pop* p = pop;
  if (count < 2) PBRL_THROW(PBRL_E_CONFIG, "cem_update: need at least 2 candidates");
  if (count % 2 != 0) PBRL_THROW(PBRL_E_CONFIG, "cem_update: candidate count must be even");
  if (count != static_cast<uint64_t>(p->n))
    PBRL_THROW(PBRL_E_CONFIG, "cem_update: scores length != candidate count");
  for (uint64_t i = 0; i < count; ++i)
    if (!std::isfinite(scores[i])) PBRL_THROW(PBRL_E_CONFIG, "cem_update: scores must be finite");
  if (!sampled) PBRL_THROW(PBRL_E_USAGE, "cem_update: no candidates sampled yet");
  std::vector<uint64_t> order(count);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](uint64_t a, uint64_t b) { return scores[a] > scores[b]; });
  const int elite = static_cast<int>(elite_fraction * static_cast<double>(count));
  if (elite < 1) PBRL_THROW(PBRL_E_CONFIG, "cem_update: elite fraction selects no candidate");
  order_d.alloc(count);
  order_d.upload(order.data(), count, p->stream);
  const int blocks = static_cast<int>(std::min<uint64_t>((dim + 255) / 256, 148 * 8));
  launch_k(k_cem_refit, std::max(blocks, 1), 256, 0, p->stream, cand.p, dim, order_d.p, elite,
           mean.p, var.p);
  p->count_launch(1);
  noise = std::max(noise_final, noise * noise_decay);
  p->sync();
}

}  // namespace pbrl
