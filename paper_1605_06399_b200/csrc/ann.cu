// ann.cu -- the auto-tuner's machine-learning performance model (§4
// lines 249-256), host code only.
//
// "the auto-tuner will execute the code of several randomly
// selected parameter configurations and record the execution times.  This
// data is then used to build an artificial neural network performance model,
// which can predict the execution time of unseen configurations.  The model is
// then used to predict the execution time of all possible configurations ...
// In a second step, some of the configurations with the best predicted
// execution times are executed, and the configuration with the best actual
// execution time of these is returned by the auto-tuner."
//
// The paper cites its earlier tuner for the network and gives no
// hyper-parameters; the fixed recipe here (R23) is SPEC.md:546-553's:
// one hidden layer of 16 tanh units, inputs and log-time targets standardised,
// weights ~ N(0,1)/sqrt(fan-in) from a seeded SplitMix64 stream, 500 epochs of
// mini-batches of 8 (seeded shuffle), step 0.01 decayed by 0.99 per epoch
// (Adam moments), mean-squared error.  Failed configurations are kept out of
// the training set.  Everything is deterministic given the seed.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <functional>
#include <numeric>
#include <vector>

#include <cstdio>

#include "internal.h"

namespace icl {

namespace {

struct Rng {  // SplitMix64
  uint64_t s;
  uint64_t next() {
    uint64_t z = (s += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  double u01() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
  double normal() {  // Box-Muller
    double u = u01(), v = u01();
    if (u < 1e-300) u = 1e-300;
    return std::sqrt(-2.0 * std::log(u)) * std::cos(6.283185307179586 * v);
  }
  uint64_t below(uint64_t n) { return next() % n; }
};

constexpr int kHidden = 16, kEpochs = 500, kBatch = 8;
constexpr double kStep = 0.01, kDecay = 0.99;

}  // namespace

struct AnnModel {
  int nf = 0;
  std::vector<double> mu, sd;  // feature standardisation
  double ymu = 0.0, ysd = 1.0; // target (log time) standardisation
  std::vector<double> W1;      // [kHidden][nf]
  std::vector<double> b1;      // [kHidden]
  std::vector<double> W2;      // [kHidden]
  double b2 = 0.0;
  double final_loss = 0.0;     // standardised MSE on the training set

  double forward(const double* xs, double* hid) const {  // xs: standardised features
    double y = b2;
    for (int j = 0; j < kHidden; ++j) {
      double a = b1[j];
      for (int f = 0; f < nf; ++f) a += W1[j * nf + f] * xs[f];
      hid[j] = std::tanh(a);
      y += W2[j] * hid[j];
    }
    return y;
  }
  double predict_log(const double* x) const {  // raw features -> predicted log value
    std::vector<double> xs(nf);
    double hid[kHidden];
    for (int f = 0; f < nf; ++f) xs[f] = (x[f] - mu[f]) / sd[f];
    return forward(xs.data(), hid) * ysd + ymu;
  }
};

// Fit the model to (X[n][nf], value[n] > 0); targets are log(value).
static void ann_fit(const double* X, const double* value, int n, int nf, uint64_t seed, AnnModel* m) {
  m->nf = nf;
  m->mu.assign(nf, 0.0);
  m->sd.assign(nf, 1.0);
  for (int f = 0; f < nf; ++f) {
    double s = 0.0, q = 0.0;
    for (int i = 0; i < n; ++i) s += X[i * nf + f];
    const double mean = s / n;
    for (int i = 0; i < n; ++i) q += (X[i * nf + f] - mean) * (X[i * nf + f] - mean);
    const double sd = std::sqrt(q / n);
    m->mu[f] = mean;
    m->sd[f] = sd > 1e-12 ? sd : 1.0;
  }
  std::vector<double> xs((size_t)n * nf), y(n);
  for (int i = 0; i < n; ++i)
    for (int f = 0; f < nf; ++f) xs[(size_t)i * nf + f] = (X[(size_t)i * nf + f] - m->mu[f]) / m->sd[f];
  double ys = 0.0, yq = 0.0;
  for (int i = 0; i < n; ++i) ys += std::log(value[i]);
  m->ymu = ys / n;
  for (int i = 0; i < n; ++i) yq += (std::log(value[i]) - m->ymu) * (std::log(value[i]) - m->ymu);
  m->ysd = std::sqrt(yq / n) > 1e-12 ? std::sqrt(yq / n) : 1.0;
  for (int i = 0; i < n; ++i) y[i] = (std::log(value[i]) - m->ymu) / m->ysd;

  Rng rng{seed ^ 0xA5A5A5A55A5A5A5Aull};
  const int P = kHidden * nf + kHidden + kHidden + 1;  // W1, b1, W2, b2 flattened
  std::vector<double> th(P, 0.0), g(P), mom(P, 0.0), vel(P, 0.0);
  for (int j = 0; j < kHidden; ++j)
    for (int f = 0; f < nf; ++f) th[j * nf + f] = rng.normal() / std::sqrt((double)nf);
  for (int j = 0; j < kHidden; ++j) th[kHidden * nf + kHidden + j] = rng.normal() / std::sqrt((double)kHidden);
  auto unpack = [&]() {
    m->W1.assign(th.begin(), th.begin() + kHidden * nf);
    m->b1.assign(th.begin() + kHidden * nf, th.begin() + kHidden * nf + kHidden);
    m->W2.assign(th.begin() + kHidden * nf + kHidden, th.begin() + kHidden * nf + 2 * kHidden);
    m->b2 = th[P - 1];
  };
  std::vector<int> order(n);
  std::iota(order.begin(), order.end(), 0);
  const double b1m = 0.9, b2m = 0.999, eps = 1e-8;
  long t = 0;
  double hid[kHidden];
  for (int ep = 0; ep < kEpochs; ++ep) {
    const double lr = kStep * std::pow(kDecay, ep);
    for (int i = n - 1; i > 0; --i) std::swap(order[i], order[rng.below((uint64_t)i + 1)]);
    for (int s0 = 0; s0 < n; s0 += kBatch) {
      const int s1 = std::min(n, s0 + kBatch);
      unpack();
      std::fill(g.begin(), g.end(), 0.0);
      for (int ii = s0; ii < s1; ++ii) {
        const int i = order[ii];
        const double* x = &xs[(size_t)i * nf];
        const double e = m->forward(x, hid) - y[i];  // d(0.5 e^2)/dy
        for (int j = 0; j < kHidden; ++j) {
          g[kHidden * nf + kHidden + j] += e * hid[j];
          const double dz = e * m->W2[j] * (1.0 - hid[j] * hid[j]);
          g[kHidden * nf + j] += dz;
          for (int f = 0; f < nf; ++f) g[j * nf + f] += dz * x[f];
        }
        g[P - 1] += e;
      }
      ++t;
      const double inv = 1.0 / (s1 - s0);
      const double c1 = 1.0 - std::pow(b1m, (double)t), c2 = 1.0 - std::pow(b2m, (double)t);
      for (int k = 0; k < P; ++k) {
        const double gk = g[k] * inv;
        mom[k] = b1m * mom[k] + (1.0 - b1m) * gk;
        vel[k] = b2m * vel[k] + (1.0 - b2m) * gk * gk;
        th[k] -= lr * (mom[k] / c1) / (std::sqrt(vel[k] / c2) + eps);
      }
    }
  }
  unpack();
  double loss = 0.0;
  for (int i = 0; i < n; ++i) {
    const double e = m->forward(&xs[(size_t)i * nf], hid) - y[i];
    loss += e * e;
  }
  m->final_loss = loss / n;
}

int ann_search(int ncfg, int nf, const double* feats, const std::function<bool(int, double*)>& evaluate, int n1,
               int topk, uint64_t seed, std::vector<int>* evaluated, int* best, double* best_val) {
  *best = -1;
  *best_val = 0.0;
  std::vector<char> done(ncfg, 0);
  std::vector<int> ok_idx;
  std::vector<double> ok_val;
  auto run = [&](int c) {
    done[c] = 1;
    if (evaluated) evaluated->push_back(c);
    double v = 0.0;
    if (!evaluate(c, &v) || !(v > 0.0) || !std::isfinite(v)) return;
    ok_idx.push_back(c);
    ok_val.push_back(v);
    if (*best < 0 || v < *best_val || (v == *best_val && c < *best)) {
      *best = c;
      *best_val = v;
    }
  };
  // phase 1: n1 distinct configurations drawn uniformly (seeded partial Fisher-Yates)
  Rng rng{seed};
  std::vector<int> perm(ncfg);
  std::iota(perm.begin(), perm.end(), 0);
  const int m1 = std::min(n1, ncfg);
  for (int i = 0; i < m1; ++i) {
    std::swap(perm[i], perm[i + (int)rng.below((uint64_t)(ncfg - i))]);
    run(perm[i]);
  }
  std::vector<int> rest;
  for (int c = 0; c < ncfg; ++c)
    if (!done[c]) rest.push_back(c);
  if (rest.empty()) return (int)ok_idx.size();
  if ((int)ok_idx.size() < kAnnMinSamples) {  // too few points for a model: finish exhaustively
    for (int c : rest) run(c);
    return (int)ok_idx.size();
  }
  // phase 2: train on the ok measurements, rank every unmeasured configuration, run the top k
  std::vector<double> X;
  for (int c : ok_idx) X.insert(X.end(), feats + (size_t)c * nf, feats + (size_t)(c + 1) * nf);
  AnnModel model;
  ann_fit(X.data(), ok_val.data(), (int)ok_idx.size(), nf, seed, &model);
  std::vector<std::pair<double, int>> ranked;
  for (int c : rest) ranked.push_back({model.predict_log(feats + (size_t)c * nf), c});
  std::sort(ranked.begin(), ranked.end());  // ascending prediction, ties -> lower index
  const int k = std::min<int>(topk, (int)ranked.size());
  for (int i = 0; i < k; ++i) run(ranked[i].second);
  return (int)ok_idx.size();
}

}  // namespace icl

// ------------------------------------------------------------------ C ABI
extern "C" {

icl_status icl_ann_fit(const double* X, const double* value, int n, int n_features, uint64_t seed, double* final_loss,
                       double* pred_value) {
  if (!X || !value || n_features < 1) return icl::report_error(ICL_ERR_INVALID_ARG, "null data or no features");
  if (n < icl::kAnnMinSamples) return icl::report_error(ICL_ERR_INVALID_ARG, "surrogate needs >= 10 samples");
  for (int i = 0; i < n; ++i)
    if (!(value[i] > 0.0) || !std::isfinite(value[i])) return icl::report_error(ICL_ERR_INVALID_ARG, "values must be > 0");
  icl::AnnModel m;
  icl::ann_fit(X, value, n, n_features, seed, &m);
  if (final_loss) *final_loss = m.final_loss;
  if (pred_value)
    for (int i = 0; i < n; ++i) pred_value[i] = std::exp(m.predict_log(X + (size_t)i * n_features));
  return ICL_OK;
}

icl_status icl_ann_search(const double* features, int n_configs, int n_features, icl_eval_fn evaluate, void* ctx,
                          int n1, int topk, uint64_t seed, int* best_index, double* best_value, int* evaluated,
                          int* n_evaluated) {
  if (!features || !evaluate || !best_index || n_configs < 1 || n_features < 1)
    return icl::report_error(ICL_ERR_INVALID_ARG, "bad ann search arguments");
  if (n1 < 1 || topk < 0) return icl::report_error(ICL_ERR_INVALID_ARG, "n1 must be >= 1 and topk >= 0");
  std::vector<int> order;
  int best = -1;
  double bv = 0.0;
  icl::ann_search(
      n_configs, n_features, features,
      [&](int c, double* v) { return evaluate(ctx, c, v) == 0; }, n1, topk, seed, &order, &best, &bv);
  if (evaluated) std::copy(order.begin(), order.end(), evaluated);
  if (n_evaluated) *n_evaluated = (int)order.size();
  *best_index = best;
  if (best_value) *best_value = bv;
  if (best < 0) return icl::report_error(ICL_ERR_UNSUPPORTED, "no configuration evaluated successfully");
  return ICL_OK;
}

}  // extern "C"
