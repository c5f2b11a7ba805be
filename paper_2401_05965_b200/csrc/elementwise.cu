// Elementwise instructions and their adjoints, plus the data-movement and
// optimizer kernels of the executor.  All are HBM-bound: 16-byte vector
// accesses when the pointers allow it, fp32 math, persistent grid capped at
// `sm_cap` CTAs of 1024 threads (one CTA per SM), grid-stride loops.
//
//   elemwise_unary   reference interpreter.py:141-143
//   elemwise_binary  reference interpreter.py:144-148
//   identity         reference interpreter.py:151-152 (a copy / axpy)
//   *_shard slicing  reference interpreter.py:81-91, 135-138 (copy_block)
#include <type_traits>

#include "common.cuh"

namespace hap {
namespace {

constexpr int kBlock = 1024;
constexpr int kUnroll = 2;   // independent 16-byte vectors in flight per thread

// Vector of 8 elements loaded/stored as one 16-byte (bf16) or two 16-byte (fp32) accesses.
template <typename T> struct Vec8;
template <> struct Vec8<__nv_bfloat16> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, float (&v)[8]) {
    uint4 raw = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x;
      v[2 * i + 1] = f.y;
    }
  }
  static __device__ __forceinline__ void store(__nv_bfloat16* p, const float (&v)[8]) {
    uint4 raw;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&raw);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = raw;
  }
};
template <> struct Vec8<float> {
  static __device__ __forceinline__ void load(const float* p, float (&v)[8]) {
    float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  static __device__ __forceinline__ void store(float* p, const float (&v)[8]) {
    reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
  }
};

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

inline int grid_for(int64_t n, int sm_cap) {
  return capped_grid((n + 8LL * kBlock - 1) / (8LL * kBlock), sm_cap);
}

// ---------------------------------------------------------------- unary
template <int tag, typename Tin, typename Tout>
__global__ void __launch_bounds__(kBlock) unary_kernel(const Tin* __restrict__ x, Tout* __restrict__ y,
                                                       int64_t n, int vec) {
  hap::pdl_enter();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (vec) {
    const int64_t nv = n / 8;
    for (int64_t base = tid; base < nv; base += kUnroll * stride) {
      float v[kUnroll][8];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (base + u * stride < nv) Vec8<Tin>::load(x + 8 * (base + u * stride), v[u]);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        if (base + u * stride >= nv) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) v[u][j] = unary_fwd(tag, v[u][j]);
        Vec8<Tout>::store(y + 8 * (base + u * stride), v[u]);
      }
    }
    for (int64_t i = nv * 8 + tid; i < n; i += stride) y[i] = from_f32<Tout>(unary_fwd(tag, to_f32(x[i])));
  } else {
    for (int64_t i = tid; i < n; i += stride) y[i] = from_f32<Tout>(unary_fwd(tag, to_f32(x[i])));
  }
}

template <int tag, typename Txy, typename Tdy, typename Tdx>
__global__ void __launch_bounds__(kBlock)
    unary_grad_kernel(const Txy* __restrict__ x, const Txy* __restrict__ y, const Tdy* __restrict__ dy,
                      Tdx* dx, int64_t n, int accumulate, int vec) {
  hap::pdl_enter();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t start = 0;
  if (vec) {  // x / y only read when the derivative needs them
    const int64_t nv = n / 8;
    const bool need_x = tag == HAP_RELU, need_y = tag != HAP_RELU && tag != HAP_NEG;
    for (int64_t base = tid; base < nv; base += kUnroll * stride) {
      float xv[kUnroll][8] = {}, yv[kUnroll][8] = {}, g[kUnroll][8], o[kUnroll][8] = {};
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t i = base + u * stride;
        if (i >= nv) continue;
        if (need_x) Vec8<Txy>::load(x + 8 * i, xv[u]);
        if (need_y) Vec8<Txy>::load(y + 8 * i, yv[u]);
        Vec8<Tdy>::load(dy + 8 * i, g[u]);
        if (accumulate) Vec8<Tdx>::load(dx + 8 * i, o[u]);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t i = base + u * stride;
        if (i >= nv) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) g[u][j] = g[u][j] * unary_deriv(tag, xv[u][j], yv[u][j]) + o[u][j];
        Vec8<Tdx>::store(dx + 8 * i, g[u]);
      }
    }
    start = nv * 8;
  }
  for (int64_t i = start + tid; i < n; i += stride) {
    const float xv = x ? to_f32(x[i]) : 0.f;
    const float yv = y ? to_f32(y[i]) : 0.f;
    float g = to_f32(dy[i]) * unary_deriv(tag, xv, yv);
    if (accumulate) g += to_f32(dx[i]);
    dx[i] = from_f32<Tdx>(g);
  }
}

// ---------------------------------------------------------------- binary
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kBlock) binary_kernel(int tag, const Tin* __restrict__ a,
                                                        const Tin* __restrict__ b,
                                                        Tout* __restrict__ out, int64_t n, int vec) {
  hap::pdl_enter();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t start = 0;
  if (vec) {
    const int64_t nv = n / 8;
    for (int64_t base = tid; base < nv; base += kUnroll * stride) {
      float va[kUnroll][8], vb[kUnroll][8];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t i = base + u * stride;
        if (i >= nv) continue;
        Vec8<Tin>::load(a + 8 * i, va[u]);
        Vec8<Tin>::load(b + 8 * i, vb[u]);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t i = base + u * stride;
        if (i >= nv) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) va[u][j] = tag == HAP_ADD ? va[u][j] + vb[u][j] : va[u][j] * vb[u][j];
        Vec8<Tout>::store(out + 8 * i, va[u]);
      }
    }
    start = nv * 8;
  }
  for (int64_t i = start + tid; i < n; i += stride) {
    const float u = to_f32(a[i]), v = to_f32(b[i]);
    out[i] = from_f32<Tout>(tag == HAP_ADD ? u + v : u * v);
  }
}

template <typename Tin, typename Tdy, typename Td>
__global__ void __launch_bounds__(kBlock)
    mul_grad_kernel(const Tin* __restrict__ a, const Tin* __restrict__ b, const Tdy* __restrict__ dy,
                    Td* da, Td* db, int64_t n, int accumulate, int vec) {
  hap::pdl_enter();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool same = da == db;
  int64_t start = 0;
  if (vec) {
    const int64_t nv = n / 8;
#pragma unroll 2
    for (int64_t i = tid; i < nv; i += stride) {
      float va[8], vb[8], g[8], ga[8], gb[8];
      Vec8<Tin>::load(a + 8 * i, va);
      Vec8<Tin>::load(b + 8 * i, vb);
      Vec8<Tdy>::load(dy + 8 * i, g);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        ga[j] = g[j] * vb[j];
        gb[j] = g[j] * va[j];
      }
      if (same && da) {
#pragma unroll
        for (int j = 0; j < 8; ++j) ga[j] += gb[j];
      }
      if (da) {
        if (accumulate) {
          float o[8];
          Vec8<Td>::load(da + 8 * i, o);
#pragma unroll
          for (int j = 0; j < 8; ++j) ga[j] += o[j];
        }
        Vec8<Td>::store(da + 8 * i, ga);
      }
      if (db && !same) {
        if (accumulate) {
          float o[8];
          Vec8<Td>::load(db + 8 * i, o);
#pragma unroll
          for (int j = 0; j < 8; ++j) gb[j] += o[j];
        }
        Vec8<Td>::store(db + 8 * i, gb);
      }
    }
    start = nv * 8;
  }
  for (int64_t i = start + tid; i < n; i += stride) {
    const float g = to_f32(dy[i]);
    const float ga = g * to_f32(b[i]), gb = g * to_f32(a[i]);
    if (same && da) {
      float v = ga + gb;
      if (accumulate) v += to_f32(da[i]);
      da[i] = from_f32<Td>(v);
    } else {
      if (da) da[i] = from_f32<Td>(accumulate ? to_f32(da[i]) + ga : ga);
      if (db) db[i] = from_f32<Td>(accumulate ? to_f32(db[i]) + gb : gb);
    }
  }
}

// ---------------------------------------------------------------- movement
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kBlock)
    axpy_kernel(float alpha, const Tin* __restrict__ x, Tout* y, int64_t n, int accumulate, int vec) {
  hap::pdl_enter();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t start = 0;
  if (vec) {
    const int64_t nv = n / 8;
    for (int64_t base = tid; base < nv; base += kUnroll * stride) {
      float v[kUnroll][8], o[kUnroll][8] = {};
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t i = base + u * stride;
        if (i >= nv) continue;
        Vec8<Tin>::load(x + 8 * i, v[u]);
        if (accumulate) Vec8<Tout>::load(y + 8 * i, o[u]);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const int64_t i = base + u * stride;
        if (i >= nv) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) v[u][j] = o[u][j] + alpha * v[u][j];
        Vec8<Tout>::store(y + 8 * i, v[u]);
      }
    }
    start = nv * 8;
  }
  for (int64_t i = start + tid; i < n; i += stride) {
    float v = alpha * to_f32(x[i]);
    if (accumulate) v += to_f32(y[i]);
    y[i] = from_f32<Tout>(v);
  }
}

// dst[o, dst_off + i, k] (+)= src[o, src_off + i, k]
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(kBlock)
    copy_block_kernel(const Tin* __restrict__ src, int64_t src_extent, int64_t src_off, Tout* dst,
                      int64_t dst_extent, int64_t dst_off, int64_t outer, int64_t count,
                      int64_t inner, int accumulate) {
  hap::pdl_enter();
  const int64_t per_outer = count * inner;
  const int64_t total = outer * per_outer;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t o = e / per_outer;
    const int64_t r = e - o * per_outer;
    const int64_t s = (o * src_extent + src_off) * inner + r;
    const int64_t d = (o * dst_extent + dst_off) * inner + r;
    float v = to_f32(src[s]);
    if (accumulate) v += to_f32(dst[d]);
    dst[d] = from_f32<Tout>(v);
  }
}

// Same-dtype block copy in VT-sized units (16, 8 or 4 bytes) when every row
// segment starts and ends on a VT boundary on both sides: the pitched copies
// of unaligned shard widths (ViT-MoE expert slices of 1804 / 1268 columns
// into 16-byte-pitched GEMM operands) moved 2 bytes per thread-iteration
// with a 64-bit division each — 31 us per 22 MB copy.
template <typename VT>
__global__ void __launch_bounds__(kBlock)
    copy_block_vec_kernel(const VT* __restrict__ src, int64_t src_row, int64_t src_off, VT* __restrict__ dst,
                          int64_t dst_row, int64_t dst_off, int64_t outer, int64_t per) {
  hap::pdl_enter();
  const int64_t total = outer * per;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total; e += stride) {
    const int64_t o = e / per;
    const int64_t r = e - o * per;
    dst[o * dst_row + dst_off + r] = src[o * src_row + src_off + r];
  }
}

template <typename T>
__global__ void fill_kernel(T* y, float value, int64_t n) {
  hap::pdl_enter();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    y[i] = from_f32<T>(value);
}

template <typename T>
__global__ void __launch_bounds__(kBlock)
    sgd_kernel(float* __restrict__ master, const float* __restrict__ grad, T* __restrict__ w,
               float lr, int64_t n) {
  hap::pdl_enter();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float v = master[i] - lr * grad[i];
    master[i] = v;
    w[i] = from_f32<T>(v);
  }
}

// Multi-tensor SGD: one launch updates every parameter tensor of the step.
// Work is split into 8192-element chunks; chunk c belongs to the tensor whose
// prefix range contains it (binary search over the chunk offsets).
struct SgdTensor {
  float* master;
  const float* grad;
  void* weight;
  int64_t n;
  int64_t first_chunk;
};

template <typename T>
__global__ void __launch_bounds__(kBlock) sgd_multi_kernel(const SgdTensor* __restrict__ ts, int count,
                                                           int64_t total_chunks, float lr) {
  hap::pdl_enter();
  constexpr int64_t kChunk = 8192;
  for (int64_t c = blockIdx.x; c < total_chunks; c += gridDim.x) {
    int lo = 0, hi = count - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ts[mid].first_chunk <= c) lo = mid; else hi = mid - 1;
    }
    const SgdTensor t = ts[lo];
    const int64_t start = (c - t.first_chunk) * kChunk;
    const int64_t end = start + kChunk < t.n ? start + kChunk : t.n;
    T* w = static_cast<T*>(t.weight);
    const bool vec = ((reinterpret_cast<uintptr_t>(t.master) | reinterpret_cast<uintptr_t>(t.grad) |
                       reinterpret_cast<uintptr_t>(w)) & 15) == 0 && (t.n % 8 == 0);
    if (vec) {
      for (int64_t i = start + 8 * threadIdx.x; i < end; i += 8 * blockDim.x) {
        float m[8], g[8];
        Vec8<float>::load(t.master + i, m);
        Vec8<float>::load(t.grad + i, g);
#pragma unroll
        for (int j = 0; j < 8; ++j) m[j] -= lr * g[j];
        Vec8<float>::store(t.master + i, m);
        Vec8<T>::store(w + i, m);
      }
    } else {
      for (int64_t i = start + threadIdx.x; i < end; i += blockDim.x) {
        const float v = t.master[i] - lr * t.grad[i];
        t.master[i] = v;
        w[i] = from_f32<T>(v);
      }
    }
  }
}

}  // namespace
}  // namespace hap

using namespace hap;

#define HAP_STREAM cudaStream_t stream = static_cast<cudaStream_t>(stream_)

extern "C" hap_status hap_unary(int tag, const void* x, hap_dtype xd, void* y, hap_dtype yd,
                                int64_t n, int sm_cap, void* stream_) {
  HAP_STREAM;
  HAP_CHECK_ARG(tag >= HAP_EXP && tag <= HAP_TANH, "hap_unary: bad tag");
  if (n <= 0) return HAP_OK;
  const int vec = aligned16(x) && aligned16(y);
  return HAP_DISPATCH_IO(xd, yd, [&] {
    auto go = [&](auto tag_c) {
      constexpr int T = decltype(tag_c)::value;
      hap::launch_k(unary_kernel<T, Tin, Tout>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream, 
          static_cast<const Tin*>(x), static_cast<Tout*>(y), n, vec);
    };
    switch (tag) {
      case HAP_EXP: go(std::integral_constant<int, HAP_EXP>{}); break;
      case HAP_NEG: go(std::integral_constant<int, HAP_NEG>{}); break;
      case HAP_RELU: go(std::integral_constant<int, HAP_RELU>{}); break;
      case HAP_SIGMOID: go(std::integral_constant<int, HAP_SIGMOID>{}); break;
      default: go(std::integral_constant<int, HAP_TANH>{}); break;
    }
    return launch_status("unary_kernel");
  });
}

extern "C" hap_status hap_unary_grad(int tag, const void* x, const void* y, hap_dtype xyd,
                                     const void* dy, hap_dtype dyd, void* dx, hap_dtype dxd,
                                     int64_t n, int accumulate, int sm_cap, void* stream_) {
  HAP_STREAM;
  HAP_CHECK_ARG(tag >= HAP_EXP && tag <= HAP_TANH, "hap_unary_grad: bad tag");
  if (n <= 0) return HAP_OK;
  HAP_CHECK_ARG(tag == HAP_NEG || (tag == HAP_RELU ? x != nullptr : y != nullptr),
                "hap_unary_grad: missing saved activation");
  const int vec = (!x || aligned16(x)) && (!y || aligned16(y)) && aligned16(dy) && aligned16(dx);
  return HAP_DISPATCH_IO(xyd, dxd, [&] {
    auto go = [&](auto tag_c) {
      constexpr int T = decltype(tag_c)::value;
      if (dyd == HAP_BF16)
        hap::launch_k(unary_grad_kernel<T, Tin, __nv_bfloat16, Tout>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream, 
            static_cast<const Tin*>(x), static_cast<const Tin*>(y), static_cast<const __nv_bfloat16*>(dy),
            static_cast<Tout*>(dx), n, accumulate, vec);
      else
        hap::launch_k(unary_grad_kernel<T, Tin, float, Tout>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream, 
            static_cast<const Tin*>(x), static_cast<const Tin*>(y), static_cast<const float*>(dy),
            static_cast<Tout*>(dx), n, accumulate, vec);
    };
    switch (tag) {
      case HAP_EXP: go(std::integral_constant<int, HAP_EXP>{}); break;
      case HAP_NEG: go(std::integral_constant<int, HAP_NEG>{}); break;
      case HAP_RELU: go(std::integral_constant<int, HAP_RELU>{}); break;
      case HAP_SIGMOID: go(std::integral_constant<int, HAP_SIGMOID>{}); break;
      default: go(std::integral_constant<int, HAP_TANH>{}); break;
    }
    return launch_status("unary_grad_kernel");
  });
}

extern "C" hap_status hap_binary(int tag, const void* a, const void* b, hap_dtype ind, void* out,
                                 hap_dtype outd, int64_t n, int sm_cap, void* stream_) {
  HAP_STREAM;
  HAP_CHECK_ARG(tag == HAP_ADD || tag == HAP_MUL, "hap_binary: bad tag");
  if (n <= 0) return HAP_OK;
  const int vec = aligned16(a) && aligned16(b) && aligned16(out);
  return HAP_DISPATCH_IO(ind, outd, [&] {
    hap::launch_k(binary_kernel<Tin, Tout>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream, 
        tag, static_cast<const Tin*>(a), static_cast<const Tin*>(b), static_cast<Tout*>(out), n, vec);
    return launch_status("binary_kernel");
  });
}

extern "C" hap_status hap_mul_grad(const void* a, const void* b, hap_dtype ind, const void* dy,
                                   hap_dtype dyd, void* da, void* db, hap_dtype dd, int64_t n,
                                   int accumulate, int sm_cap, void* stream_) {
  HAP_STREAM;
  if (n <= 0) return HAP_OK;
  const int vec = aligned16(a) && aligned16(b) && aligned16(dy) && (!da || aligned16(da)) &&
                  (!db || aligned16(db));
  return HAP_DISPATCH_IO(ind, dd, [&] {
    if (dyd == HAP_BF16)
      hap::launch_k(mul_grad_kernel<Tin, __nv_bfloat16, Tout>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream, 
          static_cast<const Tin*>(a), static_cast<const Tin*>(b),
          static_cast<const __nv_bfloat16*>(dy), static_cast<Tout*>(da), static_cast<Tout*>(db), n,
          accumulate, vec);
    else
      hap::launch_k(mul_grad_kernel<Tin, float, Tout>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream, 
          static_cast<const Tin*>(a), static_cast<const Tin*>(b), static_cast<const float*>(dy),
          static_cast<Tout*>(da), static_cast<Tout*>(db), n, accumulate, vec);
    return launch_status("mul_grad_kernel");
  });
}

extern "C" hap_status hap_axpy(float alpha, const void* x, hap_dtype xd, void* y, hap_dtype yd,
                               int64_t n, int accumulate, int sm_cap, void* stream_) {
  HAP_STREAM;
  if (n <= 0) return HAP_OK;
  const int vec = aligned16(x) && aligned16(y);
  return HAP_DISPATCH_IO(xd, yd, [&] {
    hap::launch_k(axpy_kernel<Tin, Tout>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream, 
        alpha, static_cast<const Tin*>(x), static_cast<Tout*>(y), n, accumulate, vec);
    return launch_status("axpy_kernel");
  });
}

extern "C" hap_status hap_copy_block(const void* src, hap_dtype sd, int64_t src_extent,
                                     int64_t src_off, void* dst, hap_dtype dd, int64_t dst_extent,
                                     int64_t dst_off, int64_t outer, int64_t count, int64_t inner,
                                     int accumulate, int sm_cap, void* stream_) {
  HAP_STREAM;
  HAP_CHECK_ARG(src_off >= 0 && dst_off >= 0 && src_off + count <= src_extent &&
                    dst_off + count <= dst_extent,
                "hap_copy_block: block out of range");
  const int64_t total = outer * count * inner;
  if (total <= 0) return HAP_OK;
  // Contiguous same-dtype blocks (the row shards of a leading axis) are one memcpy.
  if (outer == 1 && sd == dd && !accumulate) {
    const size_t es = dtype_size(sd);
    HAP_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(dst) + dst_off * inner * es,
                                 static_cast<const char*>(src) + src_off * inner * es,
                                 count * inner * es, cudaMemcpyDeviceToDevice, stream));
    return HAP_OK;
  }
  if (sd == dd && !accumulate) {
    const int64_t es = static_cast<int64_t>(dtype_size(sd));
    const int64_t b_src_row = src_extent * inner * es, b_dst_row = dst_extent * inner * es;
    const int64_t b_src_off = src_off * inner * es, b_dst_off = dst_off * inner * es, b_per = count * inner * es;
    auto fits = [&](int64_t v) {
      return (reinterpret_cast<uintptr_t>(src) % v) == 0 && (reinterpret_cast<uintptr_t>(dst) % v) == 0 &&
             b_src_row % v == 0 && b_dst_row % v == 0 && b_src_off % v == 0 && b_dst_off % v == 0 && b_per % v == 0;
    };
    auto launch = [&](auto tag) -> hap_status {
      using VT = decltype(tag);
      const int64_t v = sizeof(VT);
      const int64_t units = outer * (b_per / v);
      const int grid = capped_grid((units + 4LL * kBlock - 1) / (4LL * kBlock), sm_cap);
      hap::launch_k(copy_block_vec_kernel<VT>, dim3(grid), dim3(kBlock), 0, stream, static_cast<const VT*>(src),
                    b_src_row / v, b_src_off / v, static_cast<VT*>(dst), b_dst_row / v, b_dst_off / v, outer,
                    b_per / v);
      return launch_status("copy_block_vec_kernel");
    };
    if (fits(16)) return launch(uint4{});
    if (fits(8)) return launch(uint2{});
    if (fits(4)) return launch(uint32_t{});
  }
  return HAP_DISPATCH_IO(sd, dd, [&] {
    hap::launch_k(copy_block_kernel<Tin, Tout>, dim3(grid_for(total, sm_cap)), dim3(kBlock), 0, stream, 
        static_cast<const Tin*>(src), src_extent, src_off, static_cast<Tout*>(dst), dst_extent,
        dst_off, outer, count, inner, accumulate);
    return launch_status("copy_block_kernel");
  });
}

extern "C" hap_status hap_fill(void* y, hap_dtype yd, float value, int64_t n, void* stream_) {
  HAP_STREAM;
  if (n <= 0) return HAP_OK;
  const int grid = capped_grid((n + 1023) / 1024, 0);
  if (yd == HAP_BF16)
    hap::launch_k(fill_kernel<__nv_bfloat16>, dim3(grid), dim3(1024), 0, stream, static_cast<__nv_bfloat16*>(y), value, n);
  else
    hap::launch_k(fill_kernel<float>, dim3(grid), dim3(1024), 0, stream, static_cast<float*>(y), value, n);
  return launch_status("fill_kernel");
}

extern "C" hap_status hap_sgd(float* master, const float* grad, void* w, hap_dtype wd, float lr,
                              int64_t n, int sm_cap, void* stream_) {
  HAP_STREAM;
  if (n <= 0) return HAP_OK;
  if (wd == HAP_BF16)
    hap::launch_k(sgd_kernel<__nv_bfloat16>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream, 
        master, grad, static_cast<__nv_bfloat16*>(w), lr, n);
  else
    hap::launch_k(sgd_kernel<float>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream, master, grad,
                                                                  static_cast<float*>(w), lr, n);
  return launch_status("sgd_kernel");
}

extern "C" hap_status hap_sgd_multi(const void* tensors, int count, int64_t total_chunks, hap_dtype wd,
                                    float lr, int sm_cap, void* stream_) {
  HAP_STREAM;
  if (count <= 0 || total_chunks <= 0) return HAP_OK;
  const SgdTensor* ts = static_cast<const SgdTensor*>(tensors);
  const int grid = capped_grid(total_chunks, sm_cap);
  if (wd == HAP_BF16)
    hap::launch_k(sgd_multi_kernel<__nv_bfloat16>, dim3(grid), dim3(kBlock), 0, stream, ts, count, total_chunks, lr);
  else
    hap::launch_k(sgd_multi_kernel<float>, dim3(grid), dim3(kBlock), 0, stream, ts, count, total_chunks, lr);
  return launch_status("sgd_multi_kernel");
}

// ---------------------------------------------------------------- fused chains
// Elementwise chains the executor recognises in a program (all operands one
// dtype, same shape):
//   swish: y = f(x); z = x * y                    (f1 -> sigmoid -> mul)
//   gate:  p = a * b; q = f(p); o = q * c         (q*k -> sigmoid -> *v)
// Forward kernels read each input once and write every intermediate the
// program names (the backward reads them); backward kernels fuse the chain's
// adjoints and skip the gradients of the chain-internal tensors, which have
// no other consumer.
namespace hap {
namespace {

template <int tag, typename T>
__global__ void __launch_bounds__(kBlock) swish_fwd_kernel(const T* __restrict__ x, T* __restrict__ y,
                                                           T* __restrict__ z, int64_t n) {
  hap::pdl_enter();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nv = n / 8;
  for (int64_t i = tid; i < nv; i += stride) {
    float v[8], fy[8], fz[8];
    Vec8<T>::load(x + 8 * i, v);
#pragma unroll
    for (int j = 0; j < 8; ++j) fy[j] = unary_fwd(tag, v[j]);
#pragma unroll
    for (int j = 0; j < 8; j += 2) round2<T>(fy[j], fy[j + 1]);   // z uses the stored (rounded) y
#pragma unroll
    for (int j = 0; j < 8; ++j) fz[j] = v[j] * fy[j];
    Vec8<T>::store(y + 8 * i, fy);
    Vec8<T>::store(z + 8 * i, fz);
  }
  for (int64_t i = nv * 8 + tid; i < n; i += stride) {
    const float v = to_f32(x[i]);
    const T yt = from_f32<T>(unary_fwd(tag, v));
    y[i] = yt;
    z[i] = from_f32<T>(v * to_f32(yt));
  }
}

// dx (+)= dz * y + (dz * x) * f'(x, y)
template <int tag, typename T>
__global__ void __launch_bounds__(kBlock) swish_bwd_kernel(const T* __restrict__ x, const T* __restrict__ y,
                                                           const T* __restrict__ dz, T* dx, int64_t n,
                                                           int accumulate) {
  hap::pdl_enter();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nv = n / 8;
  for (int64_t i = tid; i < nv; i += stride) {
    float vx[8], vy[8], g[8], o[8] = {};
    Vec8<T>::load(x + 8 * i, vx);
    Vec8<T>::load(y + 8 * i, vy);
    Vec8<T>::load(dz + 8 * i, g);
    if (accumulate) Vec8<T>::load(dx + 8 * i, o);
    float dy[8], t[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) dy[j] = g[j] * vx[j];
#pragma unroll
    for (int j = 0; j < 8; j += 2) round2<T>(dy[j], dy[j + 1]);   // as the unfused path stores dy
#pragma unroll
    for (int j = 0; j < 8; ++j) t[j] = dy[j] * unary_deriv(tag, vx[j], vy[j]);
#pragma unroll
    for (int j = 0; j < 8; j += 2) round2<T>(t[j], t[j + 1]);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] += g[j] * vy[j] + t[j];
    Vec8<T>::store(dx + 8 * i, o);
  }
  for (int64_t i = nv * 8 + tid; i < n; i += stride) {
    const float vx = to_f32(x[i]), vy = to_f32(y[i]), g = to_f32(dz[i]);
    const float dy = to_f32(from_f32<T>(g * vx));
    float o = g * vy + to_f32(from_f32<T>(dy * unary_deriv(tag, vx, vy)));
    if (accumulate) o += to_f32(dx[i]);
    dx[i] = from_f32<T>(o);
  }
}

template <int tag, typename T>
__global__ void __launch_bounds__(kBlock) gate_fwd_kernel(const T* __restrict__ a, const T* __restrict__ b,
                                                          const T* __restrict__ c, T* __restrict__ p,
                                                          T* __restrict__ q, T* __restrict__ o, int64_t n) {
  hap::pdl_enter();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nv = n / 8;
  for (int64_t i = tid; i < nv; i += stride) {
    float va[8], vb[8], vc[8], vp[8], vq[8], vo[8];
    Vec8<T>::load(a + 8 * i, va);
    Vec8<T>::load(b + 8 * i, vb);
    Vec8<T>::load(c + 8 * i, vc);
#pragma unroll
    for (int j = 0; j < 8; ++j) vp[j] = va[j] * vb[j];
#pragma unroll
    for (int j = 0; j < 8; j += 2) round2<T>(vp[j], vp[j + 1]);
#pragma unroll
    for (int j = 0; j < 8; ++j) vq[j] = unary_fwd(tag, vp[j]);
#pragma unroll
    for (int j = 0; j < 8; j += 2) round2<T>(vq[j], vq[j + 1]);
#pragma unroll
    for (int j = 0; j < 8; ++j) vo[j] = vq[j] * vc[j];
    Vec8<T>::store(p + 8 * i, vp);
    Vec8<T>::store(q + 8 * i, vq);
    Vec8<T>::store(o + 8 * i, vo);
  }
  for (int64_t i = nv * 8 + tid; i < n; i += stride) {
    const float vp = to_f32(from_f32<T>(to_f32(a[i]) * to_f32(b[i])));
    const float vq = to_f32(from_f32<T>(unary_fwd(tag, vp)));
    p[i] = from_f32<T>(vp);
    q[i] = from_f32<T>(vq);
    o[i] = from_f32<T>(vq * to_f32(c[i]));
  }
}

// dq = do*c ; dc (+)= do*q ; dp = dq * f'(p, q) ; da (+)= dp*b ; db (+)= dp*a
template <int tag, typename T>
__global__ void __launch_bounds__(kBlock)
    gate_bwd_kernel(const T* __restrict__ a, const T* __restrict__ b, const T* __restrict__ c,
                    const T* __restrict__ p, const T* __restrict__ q, const T* __restrict__ dout, T* da, T* db,
                    T* dc, int64_t n, int acc_a, int acc_b, int acc_c) {
  hap::pdl_enter();
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nv = n / 8;
  for (int64_t i = tid; i < nv; i += stride) {   // 16-byte vectors (buffers are aligned)
    float vg[8], vq[8], vp[8], vc[8], va[8], vb[8], oa[8] = {}, ob[8] = {}, oc[8] = {};
    Vec8<T>::load(dout + 8 * i, vg);
    Vec8<T>::load(q + 8 * i, vq);
    Vec8<T>::load(p + 8 * i, vp);
    Vec8<T>::load(c + 8 * i, vc);
    Vec8<T>::load(a + 8 * i, va);
    Vec8<T>::load(b + 8 * i, vb);
    if (da && acc_a) Vec8<T>::load(da + 8 * i, oa);
    if (db && acc_b) Vec8<T>::load(db + 8 * i, ob);
    if (dc && acc_c) Vec8<T>::load(dc + 8 * i, oc);
    float dq[8], dp[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) dq[j] = vg[j] * vc[j];
#pragma unroll
    for (int j = 0; j < 8; j += 2) round2<T>(dq[j], dq[j + 1]);
#pragma unroll
    for (int j = 0; j < 8; ++j) dp[j] = dq[j] * unary_deriv(tag, vp[j], vq[j]);
#pragma unroll
    for (int j = 0; j < 8; j += 2) round2<T>(dp[j], dp[j + 1]);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      oc[j] += vg[j] * vq[j];
      oa[j] += dp[j] * vb[j];
      ob[j] += dp[j] * va[j];
    }
    if (dc) Vec8<T>::store(dc + 8 * i, oc);
    if (da) Vec8<T>::store(da + 8 * i, oa);
    if (db) Vec8<T>::store(db + 8 * i, ob);
  }
  for (int64_t i = nv * 8 + tid; i < n; i += stride) {
    const float g = to_f32(dout[i]);
    const float vq = to_f32(q[i]), vp = to_f32(p[i]);
    const float dq = to_f32(from_f32<T>(g * to_f32(c[i])));
    const float dp = to_f32(from_f32<T>(dq * unary_deriv(tag, vp, vq)));
    if (dc) dc[i] = from_f32<T>(g * vq + (acc_c ? to_f32(dc[i]) : 0.f));
    if (da) da[i] = from_f32<T>(dp * to_f32(b[i]) + (acc_a ? to_f32(da[i]) : 0.f));
    if (db) db[i] = from_f32<T>(dp * to_f32(a[i]) + (acc_b ? to_f32(db[i]) : 0.f));
  }
}

template <template <int, typename> class K, typename T>
struct TagTable;

}  // namespace
}  // namespace hap

namespace {
// Host dispatch over the unary tag for the fused kernels.
template <typename F>
hap_status with_tag(int tag, F&& f) {
  switch (tag) {
    case HAP_EXP: return f(std::integral_constant<int, HAP_EXP>{});
    case HAP_NEG: return f(std::integral_constant<int, HAP_NEG>{});
    case HAP_RELU: return f(std::integral_constant<int, HAP_RELU>{});
    case HAP_SIGMOID: return f(std::integral_constant<int, HAP_SIGMOID>{});
    default: return f(std::integral_constant<int, HAP_TANH>{});
  }
}
bool all_aligned(std::initializer_list<const void*> ps) {
  for (const void* p : ps)
    if (p && (reinterpret_cast<uintptr_t>(p) & 15)) return false;
  return true;
}
}  // namespace

extern "C" hap_status hap_swish_fwd(int tag, const void* x, void* y, void* z, hap_dtype dt, int64_t n, int sm_cap,
                                    void* stream_) {
  HAP_STREAM;
  if (n <= 0) return HAP_OK;
  HAP_CHECK_ARG(all_aligned({x, y, z}), "hap_swish_fwd: buffers must be 16-byte aligned");
  return with_tag(tag, [&](auto tc) {
    constexpr int T = decltype(tc)::value;
    if (dt == HAP_BF16)
      launch_k(swish_fwd_kernel<T, __nv_bfloat16>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream,
               static_cast<const __nv_bfloat16*>(x), static_cast<__nv_bfloat16*>(y), static_cast<__nv_bfloat16*>(z), n);
    else
      launch_k(swish_fwd_kernel<T, float>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream,
               static_cast<const float*>(x), static_cast<float*>(y), static_cast<float*>(z), n);
    return launch_status("swish_fwd_kernel");
  });
}

extern "C" hap_status hap_swish_bwd(int tag, const void* x, const void* y, const void* dz, void* dx, hap_dtype dt,
                                    int64_t n, int accumulate, int sm_cap, void* stream_) {
  HAP_STREAM;
  if (n <= 0) return HAP_OK;
  HAP_CHECK_ARG(all_aligned({x, y, dz, dx}), "hap_swish_bwd: buffers must be 16-byte aligned");
  return with_tag(tag, [&](auto tc) {
    constexpr int T = decltype(tc)::value;
    if (dt == HAP_BF16)
      launch_k(swish_bwd_kernel<T, __nv_bfloat16>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream,
               static_cast<const __nv_bfloat16*>(x), static_cast<const __nv_bfloat16*>(y),
               static_cast<const __nv_bfloat16*>(dz), static_cast<__nv_bfloat16*>(dx), n, accumulate);
    else
      launch_k(swish_bwd_kernel<T, float>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream,
               static_cast<const float*>(x), static_cast<const float*>(y), static_cast<const float*>(dz),
               static_cast<float*>(dx), n, accumulate);
    return launch_status("swish_bwd_kernel");
  });
}

extern "C" hap_status hap_gate_fwd(int tag, const void* a, const void* b, const void* c, void* p, void* q, void* o,
                                   hap_dtype dt, int64_t n, int sm_cap, void* stream_) {
  HAP_STREAM;
  if (n <= 0) return HAP_OK;
  HAP_CHECK_ARG(all_aligned({a, b, c, p, q, o}), "hap_gate_fwd: buffers must be 16-byte aligned");
  return with_tag(tag, [&](auto tc) {
    constexpr int T = decltype(tc)::value;
    if (dt == HAP_BF16) {
      using E = __nv_bfloat16;
      launch_k(gate_fwd_kernel<T, E>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream, static_cast<const E*>(a),
               static_cast<const E*>(b), static_cast<const E*>(c), static_cast<E*>(p), static_cast<E*>(q),
               static_cast<E*>(o), n);
    } else {
      launch_k(gate_fwd_kernel<T, float>, dim3(grid_for(n, sm_cap)), dim3(kBlock), 0, stream,
               static_cast<const float*>(a), static_cast<const float*>(b), static_cast<const float*>(c),
               static_cast<float*>(p), static_cast<float*>(q), static_cast<float*>(o), n);
    }
    return launch_status("gate_fwd_kernel");
  });
}

extern "C" hap_status hap_gate_bwd(int tag, const void* a, const void* b, const void* c, const void* p,
                                   const void* q, const void* dout, void* da, void* db, void* dc, hap_dtype dt,
                                   int64_t n, int acc_a, int acc_b, int acc_c, int sm_cap, void* stream_) {
  HAP_STREAM;
  if (n <= 0) return HAP_OK;
  return with_tag(tag, [&](auto tc) {
    constexpr int T = decltype(tc)::value;
    HAP_CHECK_ARG(all_aligned({a, b, c, p, q, dout, da, db, dc}), "hap_gate_bwd: buffers must be 16-byte aligned");
    const int grid = grid_for(n, sm_cap);
    if (dt == HAP_BF16) {
      using E = __nv_bfloat16;
      launch_k(gate_bwd_kernel<T, E>, dim3(grid), dim3(kBlock), 0, stream, static_cast<const E*>(a),
               static_cast<const E*>(b), static_cast<const E*>(c), static_cast<const E*>(p),
               static_cast<const E*>(q), static_cast<const E*>(dout), static_cast<E*>(da), static_cast<E*>(db),
               static_cast<E*>(dc), n, acc_a, acc_b, acc_c);
    } else {
      launch_k(gate_bwd_kernel<T, float>, dim3(grid), dim3(kBlock), 0, stream, static_cast<const float*>(a),
               static_cast<const float*>(b), static_cast<const float*>(c), static_cast<const float*>(p),
               static_cast<const float*>(q), static_cast<const float*>(dout), static_cast<float*>(da),
               static_cast<float*>(db), static_cast<float*>(dc), n, acc_a, acc_b, acc_c);
    }
    return launch_status("gate_bwd_kernel");
  });
}
