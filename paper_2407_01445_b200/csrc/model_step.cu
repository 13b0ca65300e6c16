// model_step.cu -- the model-side step AFTER the loss step: the
// reference's two-tower encoder forward / vjp (encoder.cpp:98-177; the vjp carries dE through the
// L2-normalisation Jacobian, assemble_packet engine.cpp:268-276), the gradient all-reduce
// (trainer.cpp:540-546) and the flat AdamW / LAMB optimizers (optimizers.cpp:33-63).
//
// The towers are the reference's toy linear / tanh-MLP towers in fp64 (its arithmetic); the
// matrix products run on a 16 x 16 shared-memory tiled fp64 kernel (deterministic: each output
// is one thread's fixed-order sum). The optimizer arithmetic avoids FMA contraction
// (__dmul_rn / __dadd_rn) and takes the bias corrections from the host's std::pow, so AdamW is
// bit-exact against the reference built with -ffp-contract=off; LAMB's per-layer norms are
// fixed-order block reductions (deterministic, last-bit different from a sequential sum).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <cstdint>
#include <string>

#include "../../include/fastclip_b200.h"

namespace {

thread_local std::string g_model_error;

int fail(int code, const char* msg) {
  g_model_error = msg;
  return code;
}

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return FC_OK;
  g_model_error = cudaGetErrorString(e);
  return FC_ERR_CUDA;
}

constexpr int kT = 16;

// C[m][n] (+)= sum_k A(m, k) B(k, n) with A(m, k) = A[m sam + k sak], B(k, n) = B[k sbk + n sbn];
// fixed k order per output (deterministic).
__global__ void dgemm_kernel(int M, int N, int K, const double* __restrict__ A, long long sam, long long sak,
                             const double* __restrict__ Bm, long long sbk, long long sbn, double* C, long long ldc,
                             int accumulate) {
  __shared__ double as[kT][kT + 1], bs[kT][kT + 1];
  const int m = blockIdx.y * kT + threadIdx.y, n = blockIdx.x * kT + threadIdx.x;
  double acc = 0.0;
  for (int k0 = 0; k0 < K; k0 += kT) {
    const int ka = k0 + threadIdx.x, kb = k0 + threadIdx.y;
    as[threadIdx.y][threadIdx.x] = (m < M && ka < K) ? A[m * sam + ka * sak] : 0.0;
    bs[threadIdx.y][threadIdx.x] = (kb < K && n < N) ? Bm[kb * sbk + n * sbn] : 0.0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kT; ++k) acc = __dadd_rn(acc, __dmul_rn(as[threadIdx.y][k], bs[k][threadIdx.x]));
    __syncthreads();
  }
  if (m < M && n < N) C[m * ldc + n] = accumulate ? __dadd_rn(C[m * ldc + n], acc) : acc;
}

void dgemm(cudaStream_t s, int M, int N, int K, const double* A, long long sam, long long sak, const double* Bm,
           long long sbk, long long sbn, double* C, long long ldc, bool accumulate) {
  const dim3 blk(kT, kT), grd((N + kT - 1) / kT, (M + kT - 1) / kT);
  dgemm_kernel<<<grd, blk, 0, s>>>(M, N, K, A, sam, sak, Bm, sbk, sbn, C, ldc, accumulate ? 1 : 0);
}

// z[r] += b (row broadcast), optional tanh -> h
__global__ void bias_act_kernel(double* z, const double* __restrict__ b, int rows, int cols, int act) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= static_cast<long long>(rows) * cols) return;
  double v = __dadd_rn(z[i], b[i % cols]);
  if (act) v = tanh(v);
  z[i] = v;
}

// encoder.cpp:125-132: row norms of z (|z| < 1e-12 -> NumericError), e = z / |z|, and the bf16
// copy the loss step consumes. Warp per row.
__global__ void normalize_kernel(const double* __restrict__ z, int rows, int cols, double* e, double* znorm,
                                 uint16_t* e_bf16, int* status) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
  if (r >= rows) return;
  const double* zr = z + static_cast<long long>(r) * cols;
  double ss = 0.0;
  for (int c = lane; c < cols; c += 32) ss = __dadd_rn(ss, __dmul_rn(zr[c], zr[c]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss = __dadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
  const double nrm = sqrt(ss);
  if (lane == 0) {
    znorm[r] = nrm;
    if (nrm < 1e-12) atomicCAS(status, 0, FC_ERR_NUMERIC);
  }
  for (int c = lane; c < cols; c += 32) {
    const double v = zr[c] / nrm;
    e[static_cast<long long>(r) * cols + c] = v;
    if (e_bf16) {
      const float f = static_cast<float>(v);
      uint32_t u = __float_as_uint(f);
      u += 0x7fffu + ((u >> 16) & 1u);   // round to nearest even
      e_bf16[static_cast<long long>(r) * cols + c] = static_cast<uint16_t>(u >> 16);
    }
  }
}

// encoder.cpp:151-156: cot_z = (cot - e (e . cot)) / |z| per row (warp per row).
__global__ void norm_vjp_kernel(const float* __restrict__ cot, const double* __restrict__ e,
                                const double* __restrict__ znorm, int rows, int cols, double* cz) {
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x & 31;
  if (r >= rows) return;
  const long long o = static_cast<long long>(r) * cols;
  double radial = 0.0;
  for (int c = lane; c < cols; c += 32) radial = __dadd_rn(radial, __dmul_rn(e[o + c], static_cast<double>(cot[o + c])));
#pragma unroll
  for (int k = 16; k > 0; k >>= 1) radial = __dadd_rn(radial, __shfl_xor_sync(0xffffffffu, radial, k));
  const double zn = znorm[r];
  for (int c = lane; c < cols; c += 32)
    cz[o + c] = __dadd_rn(static_cast<double>(cot[o + c]), -__dmul_rn(radial, e[o + c])) / zn;
}

// gb[c] += sum_r A[r][c] (fixed row order; thread per column)
__global__ void colsum_kernel(const double* __restrict__ A, int rows, int cols, double* gb) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  double s = 0.0;
  for (int r = 0; r < rows; ++r) s = __dadd_rn(s, A[static_cast<long long>(r) * cols + c]);
  gb[c] = __dadd_rn(gb[c], s);
}

// encoder.cpp:173: cot_a = cot_h * (1 - h^2)
__global__ void tanh_vjp_kernel(double* ch, const double* __restrict__ h, long long n) {
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) ch[i] = __dmul_rn(ch[i], 1.0 - __dmul_rn(h[i], h[i]));
}

__global__ void nonfinite_kernel(const double* __restrict__ g, long long n, int* status) {
  bool bad = false;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    bad |= !isfinite(g[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicCAS(status, 0, FC_ERR_NUMERIC);
}

struct AdamArgs {
  double b1, b2, eps, wd, lr, c1, c2;
};

// optimizers.cpp:20-30: moments and the bias-corrected direction r (no FMA contraction)
__device__ __forceinline__ double adam_dir(double& m, double& v, double g, const AdamArgs& a) {
  m = __dadd_rn(__dmul_rn(a.b1, m), __dmul_rn(1.0 - a.b1, g));
  v = __dadd_rn(__dmul_rn(a.b2, v), __dmul_rn(1.0 - a.b2, __dmul_rn(g, g)));
  return (m / a.c1) / __dadd_rn(sqrt(v / a.c2), a.eps);
}

// optimizers.cpp:33-41
__global__ void adamw_kernel(double* theta, double* m, double* v, const double* __restrict__ g, long long n, AdamArgs a,
                             const int* status) {
  if (*status) return;   // NumericError: nothing is updated (check_shapes throws first)
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double mi = m[i], vi = v[i];
    const double r = adam_dir(mi, vi, g[i], a);
    m[i] = mi;
    v[i] = vi;
    theta[i] = __dadd_rn(theta[i], -__dmul_rn(a.lr, __dadd_rn(r, __dmul_rn(a.wd, theta[i]))));
  }
}

// optimizers.cpp:43-63, first half: every moment and r (scratch), the LAMB update direction.
__global__ void lamb_dir_kernel(double* m, double* v, const double* __restrict__ g, double* r, long long n, AdamArgs a,
                                const int* status) {
  if (*status) return;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    double mi = m[i], vi = v[i];
    r[i] = adam_dir(mi, vi, g[i], a);
    m[i] = mi;
    v[i] = vi;
  }
}

// ... second half: one block per layer segment -- upd = r + wd th, trust ratio |th| / |upd|
// (1 for a zero denominator or force_alpha_one), th -= lr alpha upd. Fixed-order reductions.
__global__ void lamb_apply_kernel(double* theta, const double* __restrict__ r, const int64_t* off, const int64_t* len,
                                  AdamArgs a, int force_alpha_one, const int* status) {
  if (*status) return;
  const int64_t o = off[blockIdx.x], n = len[blockIdx.x];
  __shared__ double red[2][32];
  double st = 0.0, su = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double th = theta[o + i];
    const double u = __dadd_rn(r[o + i], __dmul_rn(a.wd, th));
    st = __dadd_rn(st, __dmul_rn(th, th));
    su = __dadd_rn(su, __dmul_rn(u, u));
  }
#pragma unroll
  for (int k = 16; k > 0; k >>= 1) {
    st = __dadd_rn(st, __shfl_xor_sync(0xffffffffu, st, k));
    su = __dadd_rn(su, __shfl_xor_sync(0xffffffffu, su, k));
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = st;
    red[1][threadIdx.x >> 5] = su;
  }
  __syncthreads();
  __shared__ double alpha;
  if (threadIdx.x == 0) {
    double t = 0.0, u = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) {
      t = __dadd_rn(t, red[0][w]);
      u = __dadd_rn(u, red[1][w]);
    }
    const double denom = sqrt(u);
    alpha = (force_alpha_one || denom == 0.0) ? 1.0 : sqrt(t) / denom;
  }
  __syncthreads();
  const double scale = __dmul_rn(a.lr, alpha);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double th = theta[o + i];
    const double u = __dadd_rn(r[o + i], __dmul_rn(a.wd, th));
    theta[o + i] = __dadd_rn(th, -__dmul_rn(scale, u));
  }
}

int grid_for(long long n) {
  long long g = (n + 255) / 256;
  return static_cast<int>(g < 1 ? 1 : (g > 4096 ? 4096 : g));
}

AdamArgs adam_args(double lr, double b1, double b2, double eps, double wd, long long step) {
  AdamArgs a{b1, b2, eps, wd, lr, 0.0, 0.0};
  a.c1 = 1.0 - std::pow(b1, static_cast<double>(step + 1));   // optimizers.cpp:22-23, host std::pow
  a.c2 = 1.0 - std::pow(b2, static_cast<double>(step + 1));
  return a;
}

}  // namespace

extern "C" {

const char* fc_model_last_error(void) { return g_model_error.c_str(); }

int fc_tower_forward(int32_t kind, int32_t rows, int32_t d_in, int32_t d_hidden, int32_t d_out, const double* theta,
                     const double* x, double* h, double* z, double* e, double* znorm, uint16_t* e_bf16,
                     int32_t* status, void* stream) {
  if (kind != 0 && kind != 1) return fail(FC_ERR_CONFIG, "tower kind must be 0 (linear) or 1 (mlp)");
  if (rows < 1 || d_in < 1 || d_out < 1 || (kind == 1 && d_hidden < 1))
    return fail(FC_ERR_CONFIG, "model: tower dims must be positive (encoder.cpp:25-30)");
  if (!theta || !x || !z || !e || !znorm || !status || (kind == 1 && !h)) return fail(FC_ERR_SHAPE, "null pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long D = d_out;
  if (kind == 0) {   // z = x W^T + b (encoder.cpp:110-113)
    dgemm(s, rows, d_out, d_in, x, d_in, 1, theta, 1, d_in, z, D, false);
    bias_act_kernel<<<grid_for(static_cast<long long>(rows) * D), 256, 0, s>>>(z, theta + D * d_in, rows, d_out, 0);
  } else {           // h = tanh(x W1^T + b1); z = h W2^T + b2 (encoder.cpp:115-123)
    const long long H = d_hidden;
    const double* w2 = theta + H * d_in + H;
    dgemm(s, rows, d_hidden, d_in, x, d_in, 1, theta, 1, d_in, h, H, false);
    bias_act_kernel<<<grid_for(static_cast<long long>(rows) * H), 256, 0, s>>>(h, theta + H * d_in, rows, d_hidden, 1);
    dgemm(s, rows, d_out, d_hidden, h, H, 1, w2, 1, H, z, D, false);
    bias_act_kernel<<<grid_for(static_cast<long long>(rows) * D), 256, 0, s>>>(z, w2 + D * H, rows, d_out, 0);
  }
  normalize_kernel<<<(rows * 32 + 255) / 256, 256, 0, s>>>(z, rows, d_out, e, znorm, e_bf16, status);
  return cuda_status(cudaGetLastError());
}

int fc_tower_vjp(int32_t kind, int32_t rows, int32_t d_in, int32_t d_hidden, int32_t d_out, const double* theta,
                 const double* x, const double* h, const double* e, const double* znorm, const float* cot,
                 double* grad, void* stream) {
  if (kind != 0 && kind != 1) return fail(FC_ERR_CONFIG, "tower kind must be 0 (linear) or 1 (mlp)");
  if (rows < 1 || d_in < 1 || d_out < 1 || (kind == 1 && d_hidden < 1))
    return fail(FC_ERR_CONFIG, "model: tower dims must be positive");
  if (!theta || !x || !e || !znorm || !cot || !grad || (kind == 1 && !h)) return fail(FC_ERR_SHAPE, "null pointer");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const long long D = d_out;
  double* cz = nullptr;
  const long long H = kind == 1 ? d_hidden : 0;
  cudaError_t ce = cudaMallocAsync(reinterpret_cast<void**>(&cz), sizeof(double) * rows * (D + H) + 8, s);
  if (ce != cudaSuccess) return cuda_status(ce);
  norm_vjp_kernel<<<(rows * 32 + 255) / 256, 256, 0, s>>>(cot, e, znorm, rows, d_out, cz);
  if (kind == 0) {   // gW += cot_z^T x, gb += colsum(cot_z) (encoder.cpp:158-163)
    dgemm(s, d_out, d_in, rows, cz, 1, D, x, d_in, 1, grad, d_in, true);
    colsum_kernel<<<(d_out + 127) / 128, 128, 0, s>>>(cz, rows, d_out, grad + D * d_in);
  } else {           // encoder.cpp:165-176
    const double* w2 = theta + H * d_in + H;
    double* gw1 = grad;
    double* gb1 = grad + H * d_in;
    double* gw2 = gb1 + H;
    double* gb2 = gw2 + D * H;
    dgemm(s, d_out, d_hidden, rows, cz, 1, D, h, H, 1, gw2, H, true);
    colsum_kernel<<<(d_out + 127) / 128, 128, 0, s>>>(cz, rows, d_out, gb2);
    double* ch = cz + static_cast<long long>(rows) * D;
    dgemm(s, rows, d_hidden, d_out, cz, D, 1, w2, H, 1, ch, H, false);   // cot_h = cot_z W2
    tanh_vjp_kernel<<<grid_for(static_cast<long long>(rows) * H), 256, 0, s>>>(ch, h, static_cast<long long>(rows) * H);
    dgemm(s, d_hidden, d_in, rows, ch, 1, H, x, d_in, 1, gw1, d_in, true);
    colsum_kernel<<<(d_hidden + 127) / 128, 128, 0, s>>>(ch, rows, d_hidden, gb1);
  }
  ce = cudaGetLastError();
  cudaFreeAsync(cz, s);
  return cuda_status(ce);
}

int fc_adamw_step(int64_t n, double* theta, double* m, double* v, int64_t* step, const double* grad, double lr,
                  double beta1, double beta2, double eps, double weight_decay, int32_t* status, void* stream) {
  if (n < 0 || !theta || !m || !v || !step || !grad || !status) return fail(FC_ERR_SHAPE, "adamw_step: bad arguments");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const AdamArgs a = adam_args(lr, beta1, beta2, eps, weight_decay, *step);
  nonfinite_kernel<<<grid_for(n), 256, 0, s>>>(grad, n, status);
  adamw_kernel<<<grid_for(n), 256, 0, s>>>(theta, m, v, grad, n, a, status);
  ++*step;   // optimizers.cpp:40 (the device status reports a rejected step)
  return cuda_status(cudaGetLastError());
}

int fc_lamb_step(int64_t n, double* theta, double* m, double* v, int64_t* step, const double* grad, double lr,
                 double beta1, double beta2, double eps, double weight_decay, int32_t n_seg, const int64_t* seg_off,
                 const int64_t* seg_len, int32_t force_alpha_one, int32_t* status, void* stream) {
  if (n < 0 || !theta || !m || !v || !step || !grad || !status) return fail(FC_ERR_SHAPE, "lamb_step: bad arguments");
  if (n_seg < 1 || !seg_off || !seg_len) return fail(FC_ERR_SHAPE, "lamb_step: layer boundaries missing");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const AdamArgs a = adam_args(lr, beta1, beta2, eps, weight_decay, *step);
  double* r = nullptr;
  int64_t* segs = nullptr;
  cudaError_t ce = cudaMallocAsync(reinterpret_cast<void**>(&r), sizeof(double) * (n + 1), s);
  if (ce == cudaSuccess) ce = cudaMallocAsync(reinterpret_cast<void**>(&segs), sizeof(int64_t) * 2 * n_seg, s);
  if (ce != cudaSuccess) return cuda_status(ce);
  cudaMemcpyAsync(segs, seg_off, sizeof(int64_t) * n_seg, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(segs + n_seg, seg_len, sizeof(int64_t) * n_seg, cudaMemcpyHostToDevice, s);
  nonfinite_kernel<<<grid_for(n), 256, 0, s>>>(grad, n, status);
  lamb_dir_kernel<<<grid_for(n), 256, 0, s>>>(m, v, grad, r, n, a, status);
  lamb_apply_kernel<<<n_seg, 256, 0, s>>>(theta, r, segs, segs + n_seg, a, force_alpha_one, status);
  ce = cudaGetLastError();
  cudaStreamSynchronize(s);   // the host segment arrays may be released by the caller on return
  cudaFreeAsync(r, s);
  cudaFreeAsync(segs, s);
  ++*step;
  return cuda_status(ce);
}

}  // extern "C"
