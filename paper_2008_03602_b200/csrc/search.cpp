// search.cpp -- model-guided candidate selection for budgets below |space|
// (host-only).
//
// The paper's tuner does not enumerate: it draws a random first batch when it
// has no data, then lets a learned cost model rank
// configurations ("machine learning based cost model ... simulated annealing",
// P:264-266) and measures the predicted-best ones, batch after batch.  The v0
// space here is small enough (<= ~1000 valid schedules per layer) that the
// model can score every unmeasured schedule, so the annealing walk is replaced
// by exhaustive scoring:
//
//   batch 0      : the first `batch` indices of the SplitMix64 sample (C17);
//   batch b > 0  : fit a ridge regression of log(latency) on the
//                  standardised schedule features over every
//                  successful measurement so far, then take the
//                  (1 - explore) * batch unmeasured schedules with the lowest
//                  prediction and fill the rest with random unmeasured ones.
//
// Deterministic given (layer, sm, measurements, seed).  Failed measurements
// (latency <= 0 or not finite) count as measured and are left out of the fit.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "tp_internal.h"

namespace tp {

static constexpr int kNF = 14;   // raw features per schedule

static double lg(double v) { return std::log2(std::max(v, 1.0)); }

// Schedule features: tile shape and pipeline knobs plus derived launch
// geometry (CTAs, k-blocks per CTA, waves at the partition's SM count, tile
// padding waste).  Kinds get indicator features.
static void features(const Layer& L, const tp_schedule& s, int sm, double* f) {
  std::fill(f, f + kNF, 0.0);
  const double ctas = (double)s.grid_x * s.grid_y * s.grid_z;
  f[6] = lg(ctas);
  f[8] = std::ceil(ctas / std::max(sm, 1));   // waves at one CTA per SM
  if (s.kind == TP_KIND_DIRECT) {
    f[0] = lg(s.threads);
    f[1] = lg(s.tile_q);
    f[2] = lg(s.vec_k);
    f[3] = lg(s.tile_p);
    f[4] = s.smem_stage;
    return;
  }
  f[0] = lg(s.bm);
  f[1] = lg(s.bn);
  f[2] = lg(s.bk);
  f[3] = s.stages;
  f[4] = s.threads / 128.0;
  f[5] = lg(s.split_k);
  int64_t kred, mext;
  if (s.kind == TP_KIND_IGEMM_TC_ROW) {
    kred = (int64_t)(L.d.c / 64) * 3;
    mext = (int64_t)L.d.n * L.P * cdiv(L.Q, s.bm) * s.bm;
    f[11] = 1.0;
    f[12] = lg(s.tiles_per_cta);
  } else if (s.kind == TP_KIND_IGEMM_TC_GATHER) {
    kred = cdiv((int64_t)L.d.r * L.d.s * L.d.c, s.bk);
    mext = cdiv(L.M, s.bm) * s.bm;
    f[13] = 1.0;
  } else {
    kred = (int64_t)L.d.r * L.d.s * cdiv(L.d.c, s.bk);
    mext = cdiv(L.M, s.bm) * s.bm;
  }
  f[7] = lg((double)kred / std::max(s.split_k, 1));
  f[9] = 1.0 - (double)L.M / (double)mext;                                   // M padding waste
  f[10] = 1.0 - (double)L.d.k / (double)(cdiv(L.d.k, s.bn) * s.bn);            // N padding waste
}

// Solve (A + lambda I) x = b for symmetric positive definite A (Cholesky).
static bool ridge_solve(std::vector<double>& A, std::vector<double>& b, int n, double lambda) {
  for (int i = 0; i < n; ++i) A[(size_t)i * n + i] += lambda;
  for (int j = 0; j < n; ++j) {
    double d = A[(size_t)j * n + j];
    for (int k = 0; k < j; ++k) d -= A[(size_t)j * n + k] * A[(size_t)j * n + k];
    if (!(d > 0)) return false;
    d = std::sqrt(d);
    A[(size_t)j * n + j] = d;
    for (int i = j + 1; i < n; ++i) {
      double v = A[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) v -= A[(size_t)i * n + k] * A[(size_t)j * n + k];
      A[(size_t)i * n + j] = v / d;
    }
  }
  for (int i = 0; i < n; ++i) {   // L y = b
    double v = b[i];
    for (int k = 0; k < i; ++k) v -= A[(size_t)i * n + k] * b[k];
    b[i] = v / A[(size_t)i * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {   // L^T x = y
    double v = b[i];
    for (int k = i + 1; k < n; ++k) v -= A[(size_t)k * n + i] * b[k];
    b[i] = v / A[(size_t)i * n + i];
  }
  return true;
}

static uint64_t smix(uint64_t& state) {
  state += 0x9E3779B97F4A7C15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace tp

using namespace tp;

extern "C" {

tp_status tp_search_next(const tp_conv_desc* d, int32_t sm_granted, const int64_t* measured_idx,
                         const double* measured_us, int32_t n_measured, int32_t batch, double explore, uint64_t seed,
                         int64_t* next_idx, int32_t* n_next) {
  Layer L;
  tp_status st = make_layer(d, &L);
  if (st != TP_OK) return st;
  if (batch < 1 || !next_idx || !n_next || n_measured < 0 || (n_measured > 0 && (!measured_idx || !measured_us)) ||
      !(explore >= 0.0 && explore <= 1.0)) {
    set_error("bad search arguments");
    return TP_EINVAL;
  }
  const std::vector<tp_schedule> space = space_all(L);
  const int64_t n = (int64_t)space.size();
  std::vector<char> done(n, 0);
  for (int32_t i = 0; i < n_measured; ++i) {
    if (measured_idx[i] < 0 || measured_idx[i] >= n) { set_error("measured index out of range"); return TP_EINVAL; }
    done[measured_idx[i]] = 1;
  }
  std::vector<int64_t> open;
  for (int64_t i = 0; i < n; ++i)
    if (!done[i]) open.push_back(i);
  const int32_t want = (int32_t)std::min<int64_t>(batch, (int64_t)open.size());
  *n_next = 0;
  if (want == 0) return TP_OK;

  // Successful measurements to fit on.
  std::vector<int32_t> ok;
  for (int32_t i = 0; i < n_measured; ++i)
    if (std::isfinite(measured_us[i]) && measured_us[i] > 0) ok.push_back(i);

  if (n_measured == 0 || ok.size() < 4) {
    // Batch 0 (or too few points to fit): the C17 sample order, skipping measured ones.
    std::vector<int64_t> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    uint64_t state = seed;
    int32_t got = 0;
    for (int64_t i = 0; i < n && got < want; ++i) {
      const int64_t j = i + (int64_t)(smix(state) % (uint64_t)(n - i));
      std::swap(perm[i], perm[j]);
      if (!done[perm[i]]) next_idx[got++] = perm[i];
    }
    *n_next = got;
    return TP_OK;
  }

  // Standardised features over the whole space.
  const int sm = std::max(1, sm_granted);
  std::vector<double> F((size_t)n * kNF);
  for (int64_t i = 0; i < n; ++i) features(L, space[i], sm, &F[(size_t)i * kNF]);
  double mu[kNF], sd[kNF];
  for (int k = 0; k < kNF; ++k) {
    double m = 0, v = 0;
    for (int64_t i = 0; i < n; ++i) m += F[(size_t)i * kNF + k];
    m /= n;
    for (int64_t i = 0; i < n; ++i) v += (F[(size_t)i * kNF + k] - m) * (F[(size_t)i * kNF + k] - m);
    mu[k] = m;
    sd[k] = v > 1e-12 ? std::sqrt(v / n) : 0.0;
  }
  // Linear model on standardised features: measured against the exhaustive
  // records (profiles/r01_search_regret.json) it ranks better than adding
  // squares or all pairwise products, which overfit the few points a small
  // budget provides.
  const int P = 1 + kNF;
  auto expand = [&](int64_t i, double* z) {
    z[0] = 1.0;
    for (int k = 0; k < kNF; ++k) z[k + 1] = sd[k] > 0 ? (F[(size_t)i * kNF + k] - mu[k]) / sd[k] : 0.0;
  };
  std::vector<double> A((size_t)P * P, 0.0), rhs(P, 0.0), z(P);
  for (int32_t r : ok) {
    expand(measured_idx[r], z.data());
    const double y = std::log(measured_us[r]);
    for (int a = 0; a < P; ++a) {
      rhs[a] += z[a] * y;
      for (int b = 0; b < P; ++b) A[(size_t)a * P + b] += z[a] * z[b];
    }
  }
  if (!ridge_solve(A, rhs, P, 1.0)) { set_error("cost-model fit failed"); return TP_EINVAL; }

  // Rank the open schedules by predicted log-latency (ties -> lowest index).
  std::vector<std::pair<double, int64_t>> pred;
  pred.reserve(open.size());
  for (int64_t i : open) {
    expand(i, z.data());
    double v = 0;
    for (int a = 0; a < P; ++a) v += z[a] * rhs[a];
    pred.emplace_back(v, i);
  }
  std::sort(pred.begin(), pred.end());
  const int32_t n_explore = std::min<int32_t>(want, (int32_t)std::lround(explore * want));
  const int32_t n_exploit = want - n_explore;
  std::vector<char> taken(n, 0);
  int32_t got = 0;
  for (int32_t k = 0; k < n_exploit; ++k) {
    next_idx[got++] = pred[k].second;
    taken[pred[k].second] = 1;
  }
  // Exploration: random open schedules not already taken, stream seeded per round.
  uint64_t state = seed ^ (0xA24BAED4963EE407ull * (uint64_t)(n_measured + 1));
  std::vector<int64_t> rest;
  for (int64_t i : open)
    if (!taken[i]) rest.push_back(i);
  for (int32_t k = 0; k < n_explore && !rest.empty(); ++k) {
    const size_t j = (size_t)(smix(state) % (uint64_t)rest.size());
    next_idx[got++] = rest[j];
    rest[j] = rest.back();
    rest.pop_back();
  }
  *n_next = got;
  return TP_OK;
}

}  // extern "C"

// Early stopping (tp.h): the last `early_stop` measured candidates did not
// strictly lower the best latency measured before them.
extern "C" int32_t tp_search_should_stop(const double* us, int32_t n, int32_t early_stop) {
  if (early_stop <= 0 || !us || n < early_stop) return 0;
  double best = -1.0;   // < 0: nothing valid measured yet
  int32_t last_improve = -1;
  for (int32_t i = 0; i < n; ++i) {
    if (us[i] >= 0.0 && (best < 0.0 || us[i] < best)) {
      best = us[i];
      last_improve = i;
    }
  }
  return (n - 1 - last_improve) >= early_stop ? 1 : 0;
}
