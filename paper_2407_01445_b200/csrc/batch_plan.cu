// batch_plan.cu -- the step BEFORE the hot path, host side: the reference's index stream
// (BatchPlan, trainer.cpp:206-241) over its deterministic RNG streams (rng.hpp:14-65), and the
// synthetic inputs SURVEY.md §8(d) derives from those streams (unit-norm bf16 embedding pairs,
// distinct ids).
//
// The generator is std::mt19937_64, which the C++ standard pins bit for bit, seeded through the
// reference's splitmix64 stream derivation; uniform / normal / below / shuffle follow rng.hpp's
// published algorithms (53-bit uniform, two-uniform Box-Muller without a cached value, rejection
// sampling, descending Fisher-Yates), so an epoch permutation here is the reference's permutation.
#include <cuda_bf16.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <initializer_list>
#include <random>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/fastclip_b200.h"

namespace {

// rng.hpp:14-19
uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// rng.hpp:23-27: stream id from a base seed and a tag list
uint64_t stream_of(uint64_t seed, std::initializer_list<uint64_t> tags) {
  uint64_t h = mix64(seed ^ 0x6a09e667f3bcc909ULL);
  for (uint64_t t : tags) h = mix64(h ^ mix64(t));
  return h;
}

struct Stream {   // rng.hpp:29-62
  std::mt19937_64 g;
  explicit Stream(uint64_t s) : g(s) {}
  double uniform() { return static_cast<double>(g() >> 11) * 0x1.0p-53; }
  double normal() {
    double u1 = uniform();
    const double u2 = uniform();
    while (u1 <= 0.0) u1 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(6.283185307179586476925286766559 * u2);
  }
  uint64_t below(uint64_t n) {
    const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
    uint64_t x = g();
    while (x >= limit) x = g();
    return x % n;
  }
  template <class T>
  void shuffle(std::vector<T>& v) {
    for (size_t i = v.size(); i > 1; --i) std::swap(v[i - 1], v[below(i)]);
  }
};

thread_local std::string g_plan_error;

struct Plan {
  int64_t n_train = 0;
  int32_t batch = 0;
  uint64_t seed = 0;
  int64_t cached_epoch = -1;
  std::vector<int32_t> perm;   // the cached epoch's permutation

  const std::vector<int32_t>& epoch_permutation(int64_t epoch) {   // trainer.cpp:216-222
    if (epoch != cached_epoch) {
      perm.resize(static_cast<size_t>(n_train));
      for (int64_t i = 0; i < n_train; ++i) perm[static_cast<size_t>(i)] = static_cast<int32_t>(i);
      Stream rng(stream_of(seed, {0x65706f6368ULL, static_cast<uint64_t>(epoch)}));
      rng.shuffle(perm);
      cached_epoch = epoch;
    }
    return perm;
  }
};

int fail(int code, const char* msg) {
  g_plan_error = msg;
  return code;
}

uint16_t to_bf16_bits(double x) {   // round to nearest even of the fp32 value
  const __nv_bfloat16 h = __float2bfloat16_rn(static_cast<float>(x));
  uint16_t b;
  std::memcpy(&b, &h, 2);
  return b;
}

}  // namespace

extern "C" {

const char* fc_plan_last_error(void) { return g_plan_error.c_str(); }

int fc_batch_plan_create(int64_t n_train, int32_t global_batch, uint64_t seed, void** plan) {
  if (!plan) return FC_ERR_SHAPE;
  *plan = nullptr;
  // BatchPlan::BatchPlan (trainer.cpp:206-214)
  if (n_train < global_batch || global_batch < 1)
    return fail(FC_ERR_CONFIG, "algo.batch_per_worker: global batch larger than the training set");
  if (n_train % global_batch != 0)
    return fail(FC_ERR_CONFIG, "algo.batch_per_worker: global batch must divide the training set");
  if (n_train > 0x7fffffffLL) return fail(FC_ERR_CONFIG, "n_train must fit int32 ids");
  auto* p = new Plan;
  p->n_train = n_train;
  p->batch = global_batch;
  p->seed = seed;
  *plan = p;
  return FC_OK;
}

int fc_batch_plan_destroy(void* plan) {
  delete static_cast<Plan*>(plan);
  return FC_OK;
}

int64_t fc_batch_plan_iters_per_epoch(void* plan) {
  const Plan* p = static_cast<const Plan*>(plan);
  return p ? p->n_train / p->batch : 0;
}

// BatchPlan::epoch_permutation (trainer.cpp:216-222): out [n_train]
int fc_batch_plan_permutation(void* plan, int64_t epoch, int32_t* out) {
  if (!plan || !out) return FC_ERR_SHAPE;
  Plan* p = static_cast<Plan*>(plan);
  const auto& perm = p->epoch_permutation(epoch);
  std::memcpy(out, perm.data(), perm.size() * sizeof(int32_t));
  return FC_OK;
}

// BatchPlan::local_batch (trainer.cpp:231-241), world = 1 / worker = 0 for the global batch
// (global_batch_indices, trainer.cpp:224-229): out [global_batch / world] in batch order.
int fc_batch_plan_local(void* plan, int64_t epoch, int64_t iter, int32_t worker, int32_t world, int32_t* out) {
  if (!plan || !out) return FC_ERR_SHAPE;
  Plan* p = static_cast<Plan*>(plan);
  if (iter < 0 || iter >= p->n_train / p->batch) return fail(FC_ERR_SHAPE, "BatchPlan: iteration out of range");
  if (world < 1 || worker < 0 || worker >= world) return fail(FC_ERR_SHAPE, "BatchPlan: bad worker");
  if (p->batch % world != 0) return fail(FC_ERR_CONFIG, "fabric.workers: worker count must divide the global batch");
  const auto& perm = p->epoch_permutation(epoch);
  const int32_t local = p->batch / world;
  std::memcpy(out, perm.data() + iter * p->batch + static_cast<int64_t>(worker) * local, local * sizeof(int32_t));
  return FC_OK;
}

// SURVEY.md §8(d) synthetic embeddings from the seed's streams: E1 = normalize(Z), Z ~ N(0, I)
// (stream {0x656d6231}); E2 = normalize(E1 + sigma N(0, I)) (stream {0x656d6232}); rows drawn in
// order, components in order; then rounded to bf16 (the oracle takes the same bf16 values).
int fc_synthetic_embeddings(uint64_t seed, int32_t rows, int32_t dim, double sigma, uint16_t* e1, uint16_t* e2) {
  if (!e1 || !e2 || rows < 0 || dim < 1) return FC_ERR_SHAPE;
  Stream r1(stream_of(seed, {0x656d6231ULL})), r2(stream_of(seed, {0x656d6232ULL}));
  std::vector<double> z(static_cast<size_t>(dim)), y(static_cast<size_t>(dim));
  for (int32_t i = 0; i < rows; ++i) {
    double n1 = 0.0;
    for (int32_t k = 0; k < dim; ++k) {
      z[k] = r1.normal();
      n1 += z[k] * z[k];
    }
    n1 = std::sqrt(n1);
    double n2 = 0.0;
    for (int32_t k = 0; k < dim; ++k) {
      z[k] /= n1;
      y[k] = z[k] + sigma * r2.normal();
      n2 += y[k] * y[k];
    }
    n2 = std::sqrt(n2);
    for (int32_t k = 0; k < dim; ++k) {
      e1[static_cast<size_t>(i) * dim + k] = to_bf16_bits(z[k]);
      e2[static_cast<size_t>(i) * dim + k] = to_bf16_bits(y[k] / n2);
    }
  }
  return FC_OK;
}

// `count` distinct ids in [0, n) by a partial Fisher-Yates over a sparse swap map with
// Rng::below (stream {0x696473}); SURVEY.md §8(d).
int fc_synthetic_ids(uint64_t seed, int32_t count, int64_t n, int32_t* ids) {
  if (!ids || count < 0 || n < count || n > 0x7fffffffLL) return FC_ERR_SHAPE;
  Stream r(stream_of(seed, {0x696473ULL}));
  std::unordered_map<int64_t, int64_t> moved;   // sparse view of the swapped prefix of iota(n)
  for (int32_t i = 0; i < count; ++i) {
    const int64_t j = i + static_cast<int64_t>(r.below(static_cast<uint64_t>(n - i)));
    const auto fi = moved.find(i), fj = moved.find(j);
    const int64_t vi = fi == moved.end() ? i : fi->second;
    const int64_t vj = fj == moved.end() ? j : fj->second;
    ids[i] = static_cast<int32_t>(vj);
    moved[j] = vi;
  }
  return FC_OK;
}

// warm u table: log10 u ~ U[-8, 0] (the paper's u percentiles,
// PAPER.md:1207-1220) from stream {0x7761726d}.
int fc_synthetic_warm_u(uint64_t seed, int64_t n, double* out) {
  if (!out || n < 0) return FC_ERR_SHAPE;
  Stream r(stream_of(seed, {0x7761726dULL}));
  for (int64_t i = 0; i < n; ++i) out[i] = std::pow(10.0, -8.0 + 8.0 * r.uniform());
  return FC_OK;
}

}  // extern "C"
