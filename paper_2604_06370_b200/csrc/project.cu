// Disaggregated projection producer (§8(f) rows f2 / f3): the step in front of the hot path that fills the two
// pools from a layer's input activations x (Eq.2; §5.1; §6 "LoRA replacement module"):
//   K_base = RoPE_t(x W_k)   V_base = x W_v          (shared bCache rows; RoPE before caching)
//   R_k    = x A_k^(a)       R_v    = x A_v^(a)      (the agent's rCache rows; RoPE deferred, P:134 / P:310)
// The base projection is a plain dense GEMM over all T rows (cuBLAS, loaded at run time); the rank-r part is a
// segmented multi-adapter product (every row its agent's A, SGMV-style) on the CUDA cores; an epilogue kernel
// rotates K at each row's absolute position and rounds the four planes into staging rows, which the row scatter
// (kv_write_kernel, control.cpp) writes into the pages.
#include <cuda_bf16.h>
#include <dlfcn.h>

#include <cstdint>
#include <mutex>
#include <string>

#include "kernels.hpp"

namespace fkv {
namespace k {
namespace {

template <typename T>
__device__ __forceinline__ float ldf(const T* p) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
  else return *reinterpret_cast<const float*>(p);
}

// R[i][0..r) = x[i] . A_k(a_i), R[i][r..2r) = x[i] . A_v(a_i): one warp per row, lanes over the hidden dimension
template <typename T, int R>
__global__ void __launch_bounds__(256) adapter_proj_kernel(const T* __restrict__ x, const int64_t* __restrict__ aptr,
                                                           int32_t n_rows, int32_t hidden, float* __restrict__ out) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (row >= n_rows) return;
  const T* ak = reinterpret_cast<const T*>(aptr[2 * row]);
  const T* av = reinterpret_cast<const T*>(aptr[2 * row + 1]);
  const T* xr = x + (int64_t)row * hidden;
  float acc[2 * R];
#pragma unroll
  for (int j = 0; j < 2 * R; ++j) acc[j] = 0.f;
  for (int h = lane; h < hidden; h += 32) {
    const float xv = ldf(xr + h);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      acc[j] += xv * ldf(ak + (int64_t)h * R + j);
      acc[R + j] += xv * ldf(av + (int64_t)h * R + j);
    }
  }
#pragma unroll
  for (int j = 0; j < 2 * R; ++j) {
    float v = acc[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    acc[j] = v;
  }
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < 2 * R; ++j) out[(int64_t)row * 2 * R + j] = acc[j];
  }
}

template <typename T>
__device__ __forceinline__ void stf(T* p, float v) {
  if constexpr (sizeof(T) == 2) *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
  else *reinterpret_cast<float*>(p) = v;
}

// Epilogue: K row (Hkv x d, fp32) rotated at the row's absolute position by the (i, i + d/2) pairs of the fp64-built
// table (C-2), V row converted, residual rows converted; block = one row, threads over the n = Hkv x d columns
template <typename T>
__global__ void __launch_bounds__(256) project_stage_kernel(const float* __restrict__ yk, const float* __restrict__ yv,
                                                            const float* __restrict__ yr, const int32_t* __restrict__ pos,
                                                            const float* __restrict__ rope_cos,
                                                            const float* __restrict__ rope_sin, int32_t hkv, int32_t d,
                                                            int32_t r, int32_t rope, T* __restrict__ kb,
                                                            T* __restrict__ vb, T* __restrict__ rk, T* __restrict__ rv) {
  const int row = blockIdx.x;
  const int n = hkv * d, half = d / 2;
  const int64_t o = (int64_t)row * n;
  const int p = pos[row];
  if (yk) {
    for (int c = threadIdx.x; c < n; c += blockDim.x) {
      const int i = c % d;
      float v = yk[o + c];
      if (rope) {
        const int j = i < half ? i : i - half;
        const float cs = rope_cos[(int64_t)p * half + j], sn = rope_sin[(int64_t)p * half + j];
        const float pair = yk[o + c + (i < half ? half : -half)];
        v = i < half ? v * cs - pair * sn : v * cs + pair * sn;
      }
      stf(kb + o + c, v);
      stf(vb + o + c, yv[o + c]);
    }
  }
  if (yr) {
    for (int c = threadIdx.x; c < r; c += blockDim.x) {
      stf(rk + (int64_t)row * r + c, yr[(int64_t)row * 2 * r + c]);
      stf(rv + (int64_t)row * r + c, yr[(int64_t)row * 2 * r + r + c]);
    }
  }
}

// ---- cuBLAS, resolved at run time (the library stays loadable on hosts without it) -----------------------------
using cublas_create_t = int (*)(void**);
using cublas_set_stream_t = int (*)(void*, cudaStream_t);
using cublas_gemm_ex_t = int (*)(void*, int, int, int, int, int, const void*, const void*, int, int, const void*, int,
                                 int, const void*, void*, int, int, int, int);
struct Blas {
  void* lib = nullptr;
  cublas_create_t create = nullptr;
  cublas_set_stream_t set_stream = nullptr;
  cublas_gemm_ex_t gemm_ex = nullptr;
  void* handle[64] = {};
  std::string err;
};
Blas& blas() {
  static Blas b;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libcublas.so.12", "/usr/local/cuda/lib64/libcublas.so.12", "libcublas.so"};
    for (const char* nm : names)
      if ((b.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!b.lib) {
      b.err = "libcublas.so.12 not found";
      return;
    }
    b.create = (cublas_create_t)dlsym(b.lib, "cublasCreate_v2");
    b.set_stream = (cublas_set_stream_t)dlsym(b.lib, "cublasSetStream_v2");
    b.gemm_ex = (cublas_gemm_ex_t)dlsym(b.lib, "cublasGemmEx");
    if (!b.create || !b.set_stream || !b.gemm_ex) b.err = "cuBLAS symbols missing";
  });
  return b;
}

}  // namespace

// Y[T][N] (fp32, row-major) = X[T][K] W[K][N] (dtype, row-major): column-major Y^T = W^T X^T
cudaError_t gemm_rowmajor_f32out(int64_t T, int64_t N, int64_t K, const void* X, const void* W, float* Y, int32_t dtype,
                                 cudaStream_t s, std::string* err) {
  Blas& b = blas();
  if (!b.err.empty()) {
    *err = b.err;
    return cudaErrorNotSupported;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!b.handle[dev] && b.create(&b.handle[dev]) != 0) {
    *err = "cublasCreate failed";
    return cudaErrorNotSupported;
  }
  void* h = b.handle[dev];
  b.set_stream(h, s);
  const float one = 1.f, zero = 0.f;
  // cudaDataType: CUDA_R_32F = 0, CUDA_R_16BF = 14; cublasComputeType_t CUBLAS_COMPUTE_32F = 68 (no TF32);
  // CUBLAS_OP_N = 0; CUBLAS_GEMM_DEFAULT = -1
  const int in_t = dtype == FKV_DTYPE_BF16 ? 14 : 0;
  const int st = b.gemm_ex(h, 0, 0, (int)N, (int)T, (int)K, &one, W, in_t, (int)N, X, in_t, (int)K, &zero, Y, 0,
                           (int)N, 68, -1);
  if (st != 0) {
    *err = "cublasGemmEx status " + std::to_string(st);
    return cudaErrorUnknown;
  }
  return cudaGetLastError();
}

cudaError_t launch_adapter_proj(const void* x, const int64_t* aptr, int32_t n_rows, int32_t hidden, int32_t r,
                                int32_t dtype, float* out, cudaStream_t s) {
  const int blocks = (n_rows * 32 + 255) / 256;
  if (n_rows <= 0) return cudaSuccess;
#define FKV_AP(R)                                                                                                    \
  if (r == R) {                                                                                                      \
    if (dtype == FKV_DTYPE_BF16)                                                                                     \
      adapter_proj_kernel<__nv_bfloat16, R><<<blocks, 256, 0, s>>>((const __nv_bfloat16*)x, aptr, n_rows, hidden, out); \
    else                                                                                                             \
      adapter_proj_kernel<float, R><<<blocks, 256, 0, s>>>((const float*)x, aptr, n_rows, hidden, out);           \
    return cudaGetLastError();                                                                                       \
  }
  FKV_AP(8)
  FKV_AP(16)
  FKV_AP(32)
  FKV_AP(64)
#undef FKV_AP
  return cudaErrorInvalidValue;
}

cudaError_t launch_project_stage(const float* yk, const float* yv, const float* yr, const int32_t* pos,
                                 const float* rope_cos, const float* rope_sin, int32_t n_rows, int32_t hkv, int32_t d,
                                 int32_t r, int32_t rope, int32_t dtype, void* kb, void* vb, void* rk, void* rv,
                                 cudaStream_t s) {
  if (n_rows <= 0) return cudaSuccess;
  if (dtype == FKV_DTYPE_BF16)
    project_stage_kernel<__nv_bfloat16><<<n_rows, 256, 0, s>>>(yk, yv, yr, pos, rope_cos, rope_sin, hkv, d, r, rope,
                                                               (__nv_bfloat16*)kb, (__nv_bfloat16*)vb,
                                                               (__nv_bfloat16*)rk, (__nv_bfloat16*)rv);
  else
    project_stage_kernel<float><<<n_rows, 256, 0, s>>>(yk, yv, yr, pos, rope_cos, rope_sin, hkv, d, r, rope,
                                                       (float*)kb, (float*)vb, (float*)rk, (float*)rv);
  return cudaGetLastError();
}

}  // namespace k
}  // namespace fkv
