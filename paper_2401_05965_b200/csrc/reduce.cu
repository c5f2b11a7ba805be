// `reduce` instruction (reference interpreter.py:149-150: np.sum over dims)
// and its adjoint (broadcast back over the reduced axes).
//
// The tensor is viewed as [outer, red, inner] when the reduced axes form one
// contiguous run — every reduction the planner emits on rank-<=2 graphs —
// with three kernels: a grid-wide sum (outer = inner = 1, e.g. the loss),
// a row sum (inner = 1) and a column sum (inner > 1, coalesced over inner and
// split over `red` across CTAs).  Accumulation is fp32 and DETERMINISTIC: a
// split reduction writes one fp32 partial per CTA into a per-stream scratch
// slot, and the last CTA to arrive (ticket counter) adds the partials in a
// fixed order — no floating-point atomics, so repeated runs give identical
// bits.  Other axis sets use a generic index-decoding kernel.
#include "common.cuh"

namespace hap {
namespace {

constexpr int kMaxRank = 8;

struct Geometry {
  int64_t outer = 1, red = 1, inner = 1;
  bool contiguous = true;
};

Geometry geometry(const int64_t* shape, int rank, uint32_t mask) {
  Geometry g;
  int first = -1, last = -1;
  for (int d = 0; d < rank; ++d)
    if (mask & (1u << d)) {
      if (first < 0) first = d;
      last = d;
    }
  if (first < 0) {  // no reduced axis: a copy
    for (int d = 0; d < rank; ++d) g.outer *= shape[d];
    return g;
  }
  for (int d = first; d <= last; ++d)
    if (!(mask & (1u << d))) g.contiguous = false;
  for (int d = 0; d < first; ++d) g.outer *= shape[d];
  for (int d = first; d <= last; ++d) g.red *= shape[d];
  for (int d = last + 1; d < rank; ++d) g.inner *= shape[d];
  return g;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float block_sum(float v) {
  __shared__ float part[32];
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) part[w] = v;
  __syncthreads();
  v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.f;
  if (w == 0) v = warp_sum(v);
  __syncthreads();
  return v;  // valid in thread 0
}

// Sum of all n elements into y[0] (+ y[0] when accumulating).  Each CTA
// writes its partial to partials[blockIdx.x]; the last CTA to take a ticket
// sums the gridDim.x partials with the fixed block_sum tree and resets the
// ticket for the next launch on the stream.
template <typename Tin>
__global__ void __launch_bounds__(1024) sum_all_kernel(const Tin* __restrict__ x, int64_t n, float* y,
                                                       int accumulate, float* partials, unsigned* ticket) {
  hap::pdl_enter();
  __shared__ bool last;
  float acc = 0.f;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    acc += to_f32(x[i]);
  acc = block_sum(acc);
  if (threadIdx.x == 0) {
    __stcg(partials + blockIdx.x, acc);
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  float v = threadIdx.x < gridDim.x ? __ldcg(partials + threadIdx.x) : 0.f;
  v = block_sum(v);
  if (threadIdx.x == 0) {
    y[0] = accumulate ? y[0] + v : v;
    *ticket = 0u;
  }
}

// One CTA per row of [outer, red]: y[o] (+)= sum_r x[o, r].
template <typename Tin, typename Tout>
__global__ void __launch_bounds__(256) row_sum_kernel(const Tin* __restrict__ x, int64_t outer,
                                                      int64_t red, Tout* y, int accumulate) {
  hap::pdl_enter();
  for (int64_t o = blockIdx.x; o < outer; o += gridDim.x) {
    float acc = 0.f;
    const Tin* row = x + o * red;
    for (int64_t r = threadIdx.x; r < red; r += blockDim.x) acc += to_f32(row[r]);
    acc = block_sum(acc);
    if (threadIdx.x == 0) y[o] = from_f32<Tout>(accumulate ? to_f32(y[o]) + acc : acc);
  }
}

// Column sums of [outer, red, inner]: CTA (bx, by) covers 256 inner
// positions of one outer slice and chunk `by` of `red`, and writes its fp32
// partial to partials[by][o * inner + i]; the last of the gridDim.y CTAs of a
// column tile (ticket per tile) adds the chunks in order into y.
template <typename Tin>
__global__ void __launch_bounds__(256) col_sum_kernel(const Tin* __restrict__ x, int64_t outer,
                                                      int64_t red, int64_t inner, int64_t chunk,
                                                      float* y, int accumulate, float* partials,
                                                      unsigned* tickets) {
  hap::pdl_enter();
  __shared__ bool last;
  const int64_t i_tiles = (inner + 255) / 256;
  const int64_t plane = outer * inner;
  for (int64_t t = blockIdx.x; t < outer * i_tiles; t += gridDim.x) {
    const int64_t o = t / i_tiles;
    const int64_t i = (t % i_tiles) * 256 + threadIdx.x;
    if (i < inner) {
      const int64_t r0 = blockIdx.y * chunk;
      const int64_t r1 = r0 + chunk < red ? r0 + chunk : red;
      float acc = 0.f;
      for (int64_t r = r0; r < r1; ++r) acc += to_f32(x[(o * red + r) * inner + i]);
      __stcg(partials + blockIdx.y * plane + o * inner + i, acc);
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(tickets + t, 1u) == gridDim.y - 1;
    __syncthreads();
    if (last) {
      __threadfence();
      if (i < inner) {
        float v = 0.f;
        for (unsigned s = 0; s < gridDim.y; ++s) v += __ldcg(partials + s * plane + o * inner + i);
        y[o * inner + i] = accumulate ? y[o * inner + i] + v : v;
      }
      if (threadIdx.x == 0) tickets[t] = 0u;
    }
    __syncthreads();
  }
}

struct Dims {
  int rank;
  int64_t shape[kMaxRank];
  uint32_t mask;
};

// Generic: thread per output element, decode kept coordinates, loop over the
// reduced coordinates.
template <typename Tin, typename Tout>
__global__ void generic_reduce_kernel(const Tin* __restrict__ x, Dims d, int64_t n_out,
                                      int64_t n_red, Tout* y, int accumulate) {
  hap::pdl_enter();
  int64_t strides[kMaxRank];
  int64_t s = 1;
  for (int a = d.rank - 1; a >= 0; --a) {
    strides[a] = s;
    s *= d.shape[a];
  }
  const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t o = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; o < n_out; o += step) {
    int64_t base = 0, rem = o;
    for (int a = d.rank - 1; a >= 0; --a)
      if (!(d.mask & (1u << a))) {
        base += (rem % d.shape[a]) * strides[a];
        rem /= d.shape[a];
      }
    float acc = 0.f;
    for (int64_t r = 0; r < n_red; ++r) {
      int64_t off = base, rr = r;
      for (int a = d.rank - 1; a >= 0; --a)
        if (d.mask & (1u << a)) {
          off += (rr % d.shape[a]) * strides[a];
          rr /= d.shape[a];
        }
      acc += to_f32(x[off]);
    }
    y[o] = from_f32<Tout>(accumulate ? to_f32(y[o]) + acc : acc);
  }
}

// Adjoint: dx[e] (+)= dy[kept coordinates of e].
template <typename Tin, typename Tout>
__global__ void unreduce_kernel(const Tin* __restrict__ dy, Dims d, Geometry g, int64_t n,
                                Tout* dx, int accumulate) {
  hap::pdl_enter();
  const int64_t step = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < n; e += step) {
    int64_t src;
    if (g.contiguous) {
      const int64_t o = e / (g.red * g.inner);
      src = o * g.inner + e % g.inner;
    } else {
      src = 0;
      int64_t rem = e, mul = 1;
      for (int a = d.rank - 1; a >= 0; --a) {
        const int64_t c = rem % d.shape[a];
        rem /= d.shape[a];
        if (!(d.mask & (1u << a))) {
          src += c * mul;
          mul *= d.shape[a];
        }
      }
    }
    float v = to_f32(dy[src]);
    if (accumulate) v += to_f32(dx[e]);
    dx[e] = from_f32<Tout>(v);
  }
}

}  // namespace
}  // namespace hap

using namespace hap;

extern "C" hap_status hap_reduce(const void* x, hap_dtype xd, const int64_t* shape, int rank,
                                 uint32_t mask, void* y, hap_dtype yd, int accumulate, int sm_cap,
                                 void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  HAP_CHECK_ARG(rank >= 0 && rank <= kMaxRank, "hap_reduce: rank > 8");
  HAP_CHECK_ARG((mask >> rank) == 0 || rank == 32, "hap_reduce: dims out of range");
  Geometry g = geometry(shape, rank, mask);
  int64_t n_out = 1;
  for (int a = 0; a < rank; ++a)
    if (!(mask & (1u << a))) n_out *= shape[a];
  if (n_out == 0) return HAP_OK;
  const size_t ysz = dtype_size(yd);
  if (g.red == 0) {  // empty reduction (zero-size shard): y = 0 (+y)
    if (!accumulate) HAP_CUDA_TRY(cudaMemsetAsync(y, 0, n_out * ysz, stream));
    return HAP_OK;
  }
  if (!g.contiguous) {
    Dims d{rank, {}, mask};
    int64_t n_red = 1;
    for (int a = 0; a < rank; ++a) {
      d.shape[a] = shape[a];
      if (mask & (1u << a)) n_red *= shape[a];
    }
    return HAP_DISPATCH_IO(xd, yd, [&] {
      hap::launch_k(generic_reduce_kernel<Tin, Tout>, dim3(capped_grid((n_out + 255) / 256, sm_cap)), dim3(256), 0, stream, 
          static_cast<const Tin*>(x), d, n_out, n_red, static_cast<Tout*>(y), accumulate);
      return launch_status("generic_reduce_kernel");
    });
  }
  if (g.inner == 1 && g.outer >= 64) {
    return HAP_DISPATCH_IO(xd, yd, [&] {
      const int rows_grid = capped_grid(g.outer, sm_cap > 0 ? 4 * sm_cap : 4 * sm_count());
      hap::launch_k(row_sum_kernel<Tin, Tout>, dim3(rows_grid), dim3(256), 0, stream, static_cast<const Tin*>(x), g.outer, g.red,
                                            static_cast<Tout*>(y), accumulate);
      return launch_status("row_sum_kernel");
    });
  }
  // Split reductions: fp32 partials in the stream's scratch, summed in order.
  HAP_CHECK_ARG(yd == HAP_F32, "hap_reduce: split reductions need an fp32 output");
  const int cap = sm_cap > 0 ? sm_cap : sm_count();
  float* partials = nullptr;
  unsigned* tickets = nullptr;
  auto scratch = [&](size_t part_floats, size_t n_tickets) -> bool {
    void* p = nullptr;
    void* t = nullptr;
    if (!stream_scratch(stream, kScratchReduce, part_floats * sizeof(float), false, &p) ||
        !stream_scratch(stream, kScratchReduceTickets, n_tickets * sizeof(unsigned), true, &t))
      return false;
    partials = static_cast<float*>(p);
    tickets = static_cast<unsigned*>(t);
    return true;
  };
  if (g.inner == 1) {  // one full sum (the loss), or a few long rows each treated as one
    const int grid = capped_grid((g.red + 4095) / 4096, cap);
    HAP_CHECK_ARG(scratch(grid, 1), "hap_reduce: no reduction scratch (first use inside stream capture?)");
    const size_t xs = dtype_size(xd);
    for (int64_t o = 0; o < g.outer; ++o) {
      const void* row = static_cast<const char*>(x) + o * g.red * xs;
      if (xd == HAP_BF16)
        hap::launch_k(sum_all_kernel<__nv_bfloat16>, dim3(grid), dim3(1024), 0, stream,
                      static_cast<const __nv_bfloat16*>(row), g.red, static_cast<float*>(y) + o, accumulate,
                      partials, tickets);
      else
        hap::launch_k(sum_all_kernel<float>, dim3(grid), dim3(1024), 0, stream, static_cast<const float*>(row),
                      g.red, static_cast<float*>(y) + o, accumulate, partials, tickets);
    }
    return launch_status("sum_all_kernel");
  }
  const int64_t i_tiles = (g.inner + 255) / 256;
  const int64_t want_y = (4LL * cap + g.outer * i_tiles - 1) / (g.outer * i_tiles);
  int64_t splits = want_y < 1 ? 1 : want_y;
  if (splits > g.red) splits = g.red;
  const int64_t chunk = (g.red + splits - 1) / splits;
  splits = (g.red + chunk - 1) / chunk;
  dim3 grid(static_cast<unsigned>(capped_grid(g.outer * i_tiles, 4 * cap)),
            static_cast<unsigned>(splits));
  HAP_CHECK_ARG(scratch(static_cast<size_t>(splits) * g.outer * g.inner, g.outer * i_tiles),
                "hap_reduce: no reduction scratch (first use inside stream capture?)");
  if (xd == HAP_BF16)
    hap::launch_k(col_sum_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, stream,
        static_cast<const __nv_bfloat16*>(x), g.outer, g.red, g.inner, chunk, static_cast<float*>(y), accumulate,
        partials, tickets);
  else
    hap::launch_k(col_sum_kernel<float>, dim3(grid), dim3(256), 0, stream, static_cast<const float*>(x), g.outer,
                  g.red, g.inner, chunk, static_cast<float*>(y), accumulate, partials, tickets);
  return launch_status("col_sum_kernel");
}

extern "C" hap_status hap_unreduce(const void* dy, hap_dtype dyd, const int64_t* shape, int rank,
                                   uint32_t mask, void* dx, hap_dtype dxd, int accumulate,
                                   int sm_cap, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  HAP_CHECK_ARG(rank >= 0 && rank <= kMaxRank, "hap_unreduce: rank > 8");
  Geometry g = geometry(shape, rank, mask);
  int64_t n = 1;
  for (int a = 0; a < rank; ++a) n *= shape[a];
  if (n == 0) return HAP_OK;
  Dims d{rank, {}, mask};
  for (int a = 0; a < rank; ++a) d.shape[a] = shape[a];
  return HAP_DISPATCH_IO(dyd, dxd, [&] {
    hap::launch_k(unreduce_kernel<Tin, Tout>, dim3(capped_grid((n + 1023) / 1024, sm_cap)), dim3(1024), 0, stream, 
        static_cast<const Tin*>(dy), d, g, n, static_cast<Tout*>(dx), accumulate);
    return launch_status("unreduce_kernel");
  });
}
