// ref_next.cpp -- TEST INFRASTRUCTURE ONLY.
//
// C-ABI access to the reference's own code for the SURVEY.md §8(f) rows next to the loss step,
// compiled unmodified from /root/reference (oracle/Makefile):
//   * state / checkpoint formats: state::UTable / IndividualTemp write+read (state.cpp:73-162)
//     and io::write_checkpoint / read_checkpoint (checkpoint.cpp:57-114);
//   * the RNG streams of the index plan (rng.hpp:14-65, header-only). BatchPlan itself lives in
//     trainer.cpp, which needs the encoder / dataset TUs this Eigen shim does not cover; its
//     three methods (trainer.cpp:216-241: iota + Rng::shuffle over the {"epoch", e} stream, then
//     contiguous slices) are restated here over the reference's own Rng;
//   * the model optimizers opt::adamw_step / lamb_step (optimizers.cpp:33-63);
//   * the reduce-scatter strategy's pieces engine::rs_partial_cotangents / rs_shard_scale
//     (engine.cpp:123-149) and the fabric's wire-cost model (fabric.cpp:18-28).
#include <cstring>
#include <fstream>
#include <numeric>
#include <sstream>
#include <vector>

#include "fastclip/checkpoint.hpp"
#include "fastclip/engine.hpp"
#include "fastclip/fabric.hpp"
#include "fastclip/optimizers.hpp"
#include "fastclip/rng.hpp"
#include "fastclip/state.hpp"

using namespace fastclip;

namespace {
Vector vec_of(const double* p, long long n) {
  Vector v(n);
  for (long long i = 0; i < n; ++i) v[i] = p[i];
  return v;
}
Matrix rows_of(const double* p, int rows, int cols) {
  Matrix m(rows, cols);
  for (int r = 0; r < rows; ++r)
    for (int c = 0; c < cols; ++c) m(r, c) = p[static_cast<size_t>(r) * cols + c];
  return m;
}
}  // namespace

extern "C" {

// UTable with the given tracks -> UTable::write; IndividualTemp (optional) -> write.
int ref_tables_write(const char* path, long long n, const double* u1, const double* u2, const double* tau1,
                     const double* tau2, double tau0, const double* m1, const double* v1, const long long* s1,
                     const double* m2, const double* v2, const long long* s2) {
  try {
    state::UTable t(static_cast<int>(n));
    t.load(vec_of(u1, n), vec_of(u2, n));
    std::ofstream os(path, std::ios::binary | std::ios::trunc);
    t.write(os);
    if (tau1) {
      // IndividualTemp has no setters: build its stream with its own writer from a read of an
      // equivalent record (the reader is the reference's, so the round trip pins the layout)
      std::stringstream ss;
      auto put = [&](const void* p, size_t k) { ss.write(static_cast<const char*>(p), static_cast<std::streamsize>(k)); };
      const std::int64_t nn = n;
      put(&nn, 8); put(tau1, 8 * n);
      put(&nn, 8); put(tau2, 8 * n);
      put(&tau0, 8);
      for (int trk = 0; trk < 2; ++trk)
        for (long long i = 0; i < n; ++i) {
          put(trk ? &m2[i] : &m1[i], 8);
          put(trk ? &v2[i] : &v1[i], 8);
          put(trk ? &s2[i] : &s1[i], 8);
        }
      state::IndividualTemp it = state::IndividualTemp::read(ss);
      it.write(os);
    }
    return os ? 0 : 10;
  } catch (...) {
    return 99;
  }
}

// UTable::read (+ IndividualTemp::read) -> host arrays.
int ref_tables_read(const char* path, long long n, int indiv, double* u1, double* u2, double* tau1, double* tau2,
                    double* tau0, double* m1, double* v1, long long* s1, double* m2, double* v2, long long* s2) {
  try {
    std::ifstream is(path, std::ios::binary);
    state::UTable t = state::UTable::read(is);
    if (t.size() != n) return 2;
    for (long long i = 0; i < n; ++i) { u1[i] = t.u1()[i]; u2[i] = t.u2()[i]; }
    if (indiv) {
      state::IndividualTemp it = state::IndividualTemp::read(is);
      for (long long i = 0; i < n; ++i) {
        tau1[i] = it.tau1()[i]; tau2[i] = it.tau2()[i];
        m1[i] = it.adam1()[i].m; v1[i] = it.adam1()[i].v; s1[i] = it.adam1()[i].step;
        m2[i] = it.adam2()[i].m; v2[i] = it.adam2()[i].v; s2[i] = it.adam2()[i].step;
      }
      *tau0 = 0.0;   // private in IndividualTemp (no accessor); the byte comparisons cover it
    }
    return 0;
  } catch (const IoError&) {
    return 10;
  } catch (...) {
    return 99;
  }
}

// io::read_checkpoint(in) -> io::write_checkpoint(out): the reference's reader and writer.
int ref_checkpoint_rewrite(const char* in, const char* out) {
  try {
    io::write_checkpoint(io::read_checkpoint(in), out);
    return 0;
  } catch (const IoError&) {
    return 10;
  } catch (...) {
    return 99;
  }
}

// Header fields and tables of a checkpoint through io::read_checkpoint.
int ref_checkpoint_fields(const char* path, unsigned long long* seed, long long* next_epoch, long long* step,
                          long long* n_params, double* tau, double* tau_m, double* tau_v, long long* tau_step,
                          int* latched, int* has_ind) {
  try {
    const io::Checkpoint ck = io::read_checkpoint(path);
    *seed = ck.seed; *next_epoch = ck.next_epoch; *step = ck.global_step;
    *n_params = ck.params.size();
    *tau = ck.tau; *tau_m = ck.tau_adam.m; *tau_v = ck.tau_adam.v; *tau_step = ck.tau_adam.step;
    *latched = ck.tau_lr_latched ? 1 : 0;
    *has_ind = ck.has_individual_temp ? 1 : 0;
    return 0;
  } catch (const IoError&) {
    return 10;
  } catch (...) {
    return 99;
  }
}

// A checkpoint written by io::write_checkpoint from the given fields (linear towers).
int ref_checkpoint_make(const char* path, unsigned long long seed, long long next_epoch, long long step,
                        int d_in, int d_out, long long n_params, const double* params, const double* om,
                        const double* ov, long long opt_step, double tau, double tau_m, double tau_v,
                        long long tau_step, int latched, long long n, const double* u1, const double* u2) {
  try {
    io::Checkpoint ck;
    ck.seed = seed; ck.next_epoch = next_epoch; ck.global_step = step;
    ck.image_shape = {enc::TowerKind::linear, d_in, 0, d_out};
    ck.text_shape = {enc::TowerKind::linear, d_in, 0, d_out};
    ck.params = vec_of(params, n_params);
    ck.opt_m = vec_of(om, n_params);
    ck.opt_v = vec_of(ov, n_params);
    ck.opt_step = opt_step;
    ck.tau = tau; ck.tau_adam.m = tau_m; ck.tau_adam.v = tau_v; ck.tau_adam.step = tau_step;
    ck.tau_lr_latched = latched != 0;
    ck.u1 = vec_of(u1, n);
    ck.u2 = vec_of(u2, n);
    ck.has_individual_temp = false;
    io::write_checkpoint(ck, path);
    return 0;
  } catch (...) {
    return 99;
  }
}

// trainer.cpp:216-241 restated over the reference's Rng / stream_seed (rng.hpp).
int ref_batch_plan_local(long long n_train, int batch, unsigned long long seed, long long epoch, long long iter,
                         int worker, int world, int* out) {
  if (n_train < batch || batch < 1 || n_train % batch != 0) return 1;
  if (iter < 0 || iter >= n_train / batch || world < 1 || worker < 0 || worker >= world || batch % world) return 2;
  std::vector<int> perm(static_cast<size_t>(n_train));
  std::iota(perm.begin(), perm.end(), 0);
  Rng rng(stream_seed(seed, {0x65706f6368ULL, static_cast<std::uint64_t>(epoch)}));
  rng.shuffle(perm);
  const int local = batch / world;
  std::memcpy(out, perm.data() + iter * batch + static_cast<long long>(worker) * local, sizeof(int) * local);
  return 0;
}

// The reference's stream primitives, for pinning the synthetic-input generator.
unsigned long long ref_stream_seed2(unsigned long long seed, unsigned long long a, unsigned long long b, int ntags) {
  return ntags == 1 ? stream_seed(seed, {a}) : stream_seed(seed, {a, b});
}
void ref_rng_normals(unsigned long long stream, long long n, double* out) {
  Rng r(stream);
  for (long long i = 0; i < n; ++i) out[i] = r.normal();
}
void ref_rng_below(unsigned long long stream, long long n, unsigned long long bound, unsigned long long* out) {
  Rng r(stream);
  for (long long i = 0; i < n; ++i) out[i] = r.below(bound - static_cast<unsigned long long>(i));
}

// opt::adamw_step / lamb_step (optimizers.cpp:33-63) on host arrays (in place).
int ref_adamw_step(long long n, double* theta, double* m, double* v, long long* step, const double* grad, double lr,
                   double b1, double b2, double eps, double wd) {
  try {
    opt::FlatAdamState st(n);
    st.m = vec_of(m, n); st.v = vec_of(v, n); st.step = *step;
    Vector th = vec_of(theta, n);
    opt::adamw_step(st, th, vec_of(grad, n), lr, {b1, b2, eps, wd});
    for (long long i = 0; i < n; ++i) { theta[i] = th[i]; m[i] = st.m[i]; v[i] = st.v[i]; }
    *step = st.step;
    return 0;
  } catch (const NumericError&) {
    return 9;
  } catch (...) {
    return 99;
  }
}
int ref_lamb_step(long long n, double* theta, double* m, double* v, long long* step, const double* grad, double lr,
                  double b1, double b2, double eps, double wd, int n_seg, const long long* seg_off,
                  const long long* seg_len, int force_alpha_one) {
  try {
    opt::FlatAdamState st(n);
    st.m = vec_of(m, n); st.v = vec_of(v, n); st.step = *step;
    Vector th = vec_of(theta, n);
    std::vector<Segment> segs;
    for (int k = 0; k < n_seg; ++k) segs.push_back({seg_off[k], seg_len[k]});
    opt::lamb_step(st, th, vec_of(grad, n), lr, {b1, b2, eps, wd}, segs, force_alpha_one != 0);
    for (long long i = 0; i < n; ++i) { theta[i] = th[i]; m[i] = st.m[i]; v[i] = st.v[i]; }
    *step = st.step;
    return 0;
  } catch (const NumericError&) {
    return 9;
  } catch (...) {
    return 99;
  }
}

// engine::rs_partial_cotangents (engine.cpp:123-144): for_e1 / for_e2 [B x d] of one worker.
int ref_rs_partials(int B, int d, const double* e1, const double* e2, const double* w1, const double* w2,
                    const double* t1, const double* t2, int lo, int cnt, double* for_e1, double* for_e2) {
  try {
    engine::PairWeights w{vec_of(w1, B), vec_of(w2, B), vec_of(t1, B), vec_of(t2, B)};
    const engine::RsPartials p = engine::rs_partial_cotangents(rows_of(e1, B, d), rows_of(e2, B, d), w, lo, cnt);
    for (int r = 0; r < B; ++r)
      for (int c = 0; c < d; ++c) {
        for_e1[static_cast<size_t>(r) * d + c] = p.for_e1(r, c);
        for_e2[static_cast<size_t>(r) * d + c] = p.for_e2(r, c);
      }
    return 0;
  } catch (...) {
    return 99;
  }
}
double ref_rs_shard_scale(int world, int local, long long batch) { return engine::rs_shard_scale(world, local, batch); }

// fabric.cpp:18-28 wire-cost model.
unsigned long long ref_wire(int primitive, int world, unsigned long long payload) {
  switch (primitive) {
    case 0: return dist::all_gather_wire(world, payload);
    case 1: return dist::all_reduce_wire(world, payload);
    default: return dist::reduce_scatter_wire(world, payload);
  }
}

}  // extern "C"
