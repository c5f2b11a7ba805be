// Variable-chunk all-gather / reduce-scatter over NVLink peer memory.
//
// The reference's collectives (interpreter.py:69-101) concatenate / sum
// per-device shards whose extents come from the ratio-rounded shard table —
// uneven, possibly zero, and along any axis.  NCCL needs equal counts
// (padding to the largest shard, the cost model's all_gather) or
// pack/unpack passes for non-leading axes.  This kernel instead reads every
// peer's shard straight out of its HBM through the NVSwitch (CUDA IPC mapped
// pointers) and writes it at its final [outer, offset, inner] position:
// exact bytes, no padding, no staging pass on the receiver.
//
// Protocol per call, for rank r with peers p (all ranks run the same call):
//   1. wait until every peer has finished reading r's staging buffer from the
//      previous call (done[p] >= epoch on r's signal page);
//   2. copy r's shard into r's symmetric staging buffer (grid-stride), grid
//      barrier, then one thread publishes ready[r] = epoch+1 on every peer's
//      signal page (system-scope release);
//   3. every CTA waits for ready[p] == epoch+1 (acquire) and pulls the peers'
//      chunks over NVLink into the output (the own chunk from local staging);
//   4. grid barrier, then done[r] = epoch+1 on every peer; epoch advances in
//      device memory so CUDA-graph replays need no host bookkeeping.
// Every CTA spins on flags another GPU writes, so the grid is one CTA per
// (capped) SM, all resident; separate GPUs run the ranks, never one GPU.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <utility>
#include <string>
#include <vector>

#include "common.cuh"

namespace hap {
namespace {

constexpr int kMaxRanks = 16;
constexpr int kThreads = 512;

struct SignalPage {       // lives at the start of each rank's symmetric arena
  uint64_t ready[kMaxRanks];
  uint64_t done[kMaxRanks];
  uint64_t armed[kMaxRanks];   // push gather: peer p's output may be overwritten for call armed[p]-1
  uint64_t epoch;         // calls completed by this rank
  uint32_t arrive;        // grid-barrier counter (local)
  uint32_t generation;    // grid-barrier generation (local)
  uint64_t pad[5];
};
static_assert(sizeof(SignalPage) <= 512, "signal page too large");
constexpr size_t kSignalBytes = 512;

struct Symm {
  int rank = 0, nranks = 1;
  size_t bytes = 0;
  char* local = nullptr;                 // arena base (signal page + staging)
  char* peers[kMaxRanks] = {};           // peer arena bases (IPC-mapped), peers[rank] = local
  // (peer, IPC handle of its allocation) -> mapped here.  Keyed by the handle,
  // not the allocation's base address: a peer may free an allocation and get
  // a new one at the same address, and a mapping cached by address would
  // then point at the old memory (pushes silently lost — seen in
  // tools/coll_fit.py's all-to-all check at 2 GPUs)
  std::map<std::pair<int, std::string>, char*> opened;
  bool local_open = false;               // peers are arenas of this process (hap_symm_open_local)
};

struct Peers {
  char* base[kMaxRanks];
  // HAP_P2P_NOSYNC=1 (measurement only, results undefined): skip the waits
  // on peers' flags, so each kernel moves its NVLink bytes alone — what an
  // ncu capture of the NVLink counters needs, since ncu serialises kernels
  // and a kernel waiting for its partner would never finish under it
  int nosync;
};

int p2p_nosync() {
  static int on = [] {
    const char* v = getenv("HAP_P2P_NOSYNC");
    return v ? atoi(v) : 0;
  }();
  return on;
}

__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// All CTAs of the (fully resident) grid meet; returns true in exactly one CTA
// (the last to arrive), after which everyone proceeds.
__device__ bool grid_barrier(SignalPage* sig) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t gen = *reinterpret_cast<volatile uint32_t*>(&sig->generation);
    __threadfence();
    const uint32_t n = atomicAdd(&sig->arrive, 1u) + 1;
    last = n == gridDim.x;
    if (last) {
      sig->arrive = 0;
      __threadfence();
      atomicAdd(&sig->generation, 1u);
    } else {
      while (*reinterpret_cast<volatile uint32_t*>(&sig->generation) == gen) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
  return last;
}

template <typename T>
__device__ void copy_elems(T* __restrict__ dst, const T* __restrict__ src, int64_t n) {
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) == 0;
  if (vec) {
    constexpr int per = 16 / sizeof(T);
    const int64_t nv = n / per;
    const int4* s4 = reinterpret_cast<const int4*>(src);
    int4* d4 = reinterpret_cast<int4*>(dst);
    // 8 independent 16-byte loads in flight per thread: a peer read over
    // NVLink costs ~2 us, so bandwidth needs many outstanding requests.
    constexpr int U = 8;
    int64_t i = tid;
    for (; i + (U - 1) * stride < nv; i += U * stride) {
      int4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = s4[i + u * stride];
#pragma unroll
      for (int u = 0; u < U; ++u) d4[i + u * stride] = v[u];
    }
    for (; i < nv; i += stride) d4[i] = s4[i];
    for (int64_t j = nv * per + tid; j < n; j += stride) dst[j] = src[j];
  } else {
    for (int64_t i = tid; i < n; i += stride) dst[i] = src[i];
  }
}

// Block placement: chunk [outer, rows, inner] -> out[outer, off + rows, inner].
template <typename T>
__device__ void place_chunk(T* __restrict__ out, const T* __restrict__ chunk, int64_t outer, int64_t rows,
                            int64_t inner, int64_t extent, int64_t off) {
  if (outer == 1) {
    copy_elems(out + off * inner, chunk, rows * inner);
    return;
  }
  const int64_t per = rows * inner;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  constexpr int kv = 16 / sizeof(T);
  if (inner % kv == 0 && ((reinterpret_cast<uintptr_t>(out) | reinterpret_cast<uintptr_t>(chunk)) & 15) == 0) {
    // every [rows, inner] block starts 16-byte aligned: 16-byte moves
    const int64_t per4 = per / kv, total4 = outer * per4;
    const int4* c4 = reinterpret_cast<const int4*>(chunk);
    for (int64_t e = tid; e < total4; e += stride) {
      const int64_t o = e / per4, rem = e - o * per4;
      reinterpret_cast<int4*>(out + (o * extent + off) * inner)[rem] = c4[e];
    }
    return;
  }
  const int64_t total = outer * per;
  for (int64_t e = tid; e < total; e += stride) {
    const int64_t o = e / per, rem = e - o * per;
    out[(o * extent + off) * inner + rem] = chunk[e];
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) p2p_all_gather_kernel(Peers peers, int rank, int nranks,
                                                                  const T* __restrict__ send, T* __restrict__ out,
                                                                  int64_t outer, int64_t inner, int64_t extent,
                                                                  const int64_t* __restrict__ sizes,
                                                                  const int64_t* __restrict__ offs) {
  hap::pdl_wait();
  SignalPage* sig = reinterpret_cast<SignalPage*>(peers.base[rank]);
  T* staging = reinterpret_cast<T*>(peers.base[rank] + kSignalBytes);
  const uint64_t epoch = *reinterpret_cast<volatile uint64_t*>(&sig->epoch);
  // 1. peers have finished reading my staging buffer from the previous call
  if (threadIdx.x < nranks && threadIdx.x != rank)
    if (!peers.nosync) while (ld_acquire_sys(&sig->done[threadIdx.x]) < epoch) __nanosleep(128);
  __syncthreads();
  // 2. publish my shard
  const int64_t mine = outer * sizes[rank] * inner;
  copy_elems(staging, send, mine);
  if (grid_barrier(sig) && threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      SignalPage* peer_sig = reinterpret_cast<SignalPage*>(peers.base[p]);
      st_release_sys(&peer_sig->ready[rank], epoch + 1);
    }
  }
  // 3. pull every chunk into place
  if (threadIdx.x < nranks && threadIdx.x != rank)
    if (!peers.nosync) while (ld_acquire_sys(&sig->ready[threadIdx.x]) < epoch + 1) __nanosleep(64);
  __syncthreads();
  for (int q = 0; q < nranks; ++q) {
    const int p = (rank + q) % nranks;  // stagger sources across ranks
    // own chunk from `send` (staging was written by other CTAs of this grid
    // and could be stale in this SM's L1); peers' staging over NVLink
    const T* src = p == rank ? send : reinterpret_cast<const T*>(peers.base[p] + kSignalBytes);
    place_chunk(out, src, outer, sizes[p], inner, extent, offs[p]);
  }
  // 4. done reading the peers' staging buffers
  if (grid_barrier(sig) && threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      SignalPage* peer_sig = reinterpret_cast<SignalPage*>(peers.base[p]);
      st_release_sys(&peer_sig->done[rank], epoch + 1);
    }
    sig->epoch = epoch + 1;
  }
}

// Push all-gather into registered outputs: every rank's output buffer is
// mapped into every peer (hap_p2p_buffer_handle / _open), so rank r stores
// its shard straight into every output at its final [outer, off_r, inner]
// position — NVLink writes are posted (no request round trip), measured
// 680 GB/s per rank vs 640 for reads (tools/coll_bench.py --probe), and
// there is no staging copy.  Protocol per call (epoch e on every rank):
//   1. armed: at kernel start my stream has finished every earlier reader of
//      my output, so CTA 0 tells each peer armed[r] = e+1; every CTA waits
//      for armed[p] = e+1 before storing into p's output;
//   2. store my shard into all outputs (own included), grid barrier;
//   3. ready[r] = e+1 (and done[r], so a later staged call's reuse check
//      passes) on every peer, system-scope release; every CTA waits for
//      every peer's ready before the kernel ends, so the output is complete
//      for the next kernel on the stream.
template <typename T>
__global__ void __launch_bounds__(kThreads) p2p_all_gather_push_kernel(Peers peers, int rank, int nranks,
                                                                       const T* __restrict__ send,
                                                                       T* const* __restrict__ outs, int64_t outer,
                                                                       int64_t inner, int64_t extent,
                                                                       const int64_t* __restrict__ sizes,
                                                                       const int64_t* __restrict__ offs) {
  hap::pdl_wait();
  SignalPage* sig = reinterpret_cast<SignalPage*>(peers.base[rank]);
  const uint64_t epoch = *reinterpret_cast<volatile uint64_t*>(&sig->epoch);
  const bool peer_thread = threadIdx.x < nranks && threadIdx.x != rank;
  if (blockIdx.x == 0 && peer_thread)
    st_release_sys(&reinterpret_cast<SignalPage*>(peers.base[threadIdx.x])->armed[rank], epoch + 1);
  if (peer_thread)
    if (!peers.nosync) while (ld_acquire_sys(&sig->armed[threadIdx.x]) < epoch + 1) __nanosleep(64);
  __syncthreads();
  for (int q = 1; q <= nranks; ++q) {
    const int p = (rank + q) % nranks;   // peers staggered across ranks, own output last (local HBM)
    place_chunk(outs[p], send, outer, sizes[rank], inner, extent, offs[rank]);
  }
  if (grid_barrier(sig) && threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      SignalPage* peer_sig = reinterpret_cast<SignalPage*>(peers.base[p]);
      st_release_sys(&peer_sig->ready[rank], epoch + 1);
      st_release_sys(&peer_sig->done[rank], epoch + 1);
    }
    sig->epoch = epoch + 1;
  }
  if (peer_thread)
    if (!peers.nosync) while (ld_acquire_sys(&sig->ready[threadIdx.x]) < epoch + 1) __nanosleep(64);
}

// Reduce-scatter: rank r stages its whole partial tensor [outer, extent,
// inner]; every rank then sums, for its own shard rows, the matching rows of
// all peers' partial tensors over NVLink.
template <typename T>
__global__ void __launch_bounds__(kThreads) p2p_reduce_scatter_kernel(Peers peers, int rank, int nranks,
                                                                      const T* __restrict__ send,
                                                                      T* __restrict__ out, int64_t outer,
                                                                      int64_t inner, int64_t extent,
                                                                      const int64_t* __restrict__ sizes,
                                                                      const int64_t* __restrict__ offs) {
  hap::pdl_wait();
  SignalPage* sig = reinterpret_cast<SignalPage*>(peers.base[rank]);
  T* staging = reinterpret_cast<T*>(peers.base[rank] + kSignalBytes);
  const uint64_t epoch = *reinterpret_cast<volatile uint64_t*>(&sig->epoch);
  if (threadIdx.x < nranks && threadIdx.x != rank)
    if (!peers.nosync) while (ld_acquire_sys(&sig->done[threadIdx.x]) < epoch) __nanosleep(128);
  __syncthreads();
  copy_elems(staging, send, outer * extent * inner);
  if (grid_barrier(sig) && threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      st_release_sys(&reinterpret_cast<SignalPage*>(peers.base[p])->ready[rank], epoch + 1);
    }
  }
  if (threadIdx.x < nranks && threadIdx.x != rank)
    if (!peers.nosync) while (ld_acquire_sys(&sig->ready[threadIdx.x]) < epoch + 1) __nanosleep(64);
  __syncthreads();
  const int64_t rows = sizes[rank], off = offs[rank];
  const int64_t per = rows * inner, total = outer * per;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = tid; e < total; e += stride) {
    const int64_t o = e / per, rem = e - o * per;
    const int64_t at = (o * extent + off) * inner + rem;
    float acc = 0.f;
    for (int p = 0; p < nranks; ++p)   // rank order: the sum LocalGroup and every other path computes
      acc += to_f32(p == rank ? send[at] : reinterpret_cast<const T*>(peers.base[p] + kSignalBytes)[at]);
    out[e] = from_f32<T>(acc);
  }
  if (grid_barrier(sig) && threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      st_release_sys(&reinterpret_cast<SignalPage*>(peers.base[p])->done[rank], epoch + 1);
    }
    sig->epoch = epoch + 1;
  }
}

// Bandwidth probe (tools/coll_bench.py --probe; no flags, the caller
// separates calls with a host barrier).  Arena layout: chunk q at
// kSignalBytes + q * chunk on every rank.  Modes: 0 pull peers one after
// another, 1 push one after another, 2 pull with the grid split across peers
// (all peers at once), 3 push split across peers, 4 local copy of the same
// bytes (HBM reference).
__global__ void __launch_bounds__(kThreads) p2p_probe_kernel(Peers peers, int rank, int nranks, int mode,
                                                             int64_t chunk) {
  char* local = peers.base[rank] + kSignalBytes;
  const int64_t n4 = chunk / 16;
  if (mode == 4) {
    for (int q = 1; q < nranks; ++q)
      copy_elems(reinterpret_cast<int4*>(local + ((rank + q) % nranks) * chunk),
                 reinterpret_cast<const int4*>(local + rank * chunk), n4);
    return;
  }
  const bool push = mode == 1 || mode == 3;
  auto src_of = [&](int p) {
    return push ? reinterpret_cast<const int4*>(local + rank * chunk)
                : reinterpret_cast<const int4*>(peers.base[p] + kSignalBytes + rank * chunk);
  };
  auto dst_of = [&](int p) {
    return push ? reinterpret_cast<int4*>(peers.base[p] + kSignalBytes + rank * chunk)
                : reinterpret_cast<int4*>(local + p * chunk);
  };
  if (mode <= 1) {
    for (int q = 1; q < nranks; ++q) copy_elems(dst_of((rank + q) % nranks), src_of((rank + q) % nranks), n4);
    return;
  }
  // split: CTA b serves peer (rank + 1 + b % (nranks-1)) % nranks, striding over that peer's CTAs
  const int peers_n = nranks - 1;
  const int which = blockIdx.x % peers_n;
  const int p = (rank + 1 + which) % nranks;
  const int ctas = (gridDim.x - which + peers_n - 1) / peers_n;
  const int idx = blockIdx.x / peers_n;
  const int4* src = src_of(p);
  int4* dst = dst_of(p);
  constexpr int U = 8;
  const int64_t stride = static_cast<int64_t>(ctas) * blockDim.x;
  int64_t i = static_cast<int64_t>(idx) * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n4; i += stride) dst[i] = src[i];
}

// Reduce-scatter straight out of registered partials: every rank's partial
// tensor is mapped into every peer, so rank r sums its own shard rows from
// all partials over NVLink with no staging copy.  Per call (epoch e):
//   1. CTA 0 tells each peer ready[r] = e+1 (my partial is complete: the
//      kernel started after its producers); every CTA waits for all peers;
//   2. sum: 16-byte loads from every rank's partial (own from local HBM),
//      fp32 accumulation in rank order (0, 1, ..., m-1 — the order of the
//      single-GPU LocalGroup sum, so both give the same bits), one rounding;
//   3. grid barrier, done[r] = e+1 on every peer (finished reading theirs);
//      every CTA waits for every peer's done, so my partial is not
//      overwritten by later work on my stream while a peer still reads it.
template <typename T>
__device__ __forceinline__ void add8(float* acc, const int4& v) {
  if constexpr (sizeof(T) == 2) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      acc[2 * i] += f.x;
      acc[2 * i + 1] += f.y;
    }
  } else {
    const float* f = reinterpret_cast<const float*>(&v);
#pragma unroll
    for (int i = 0; i < 4; ++i) acc[i] += f[i];
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) p2p_reduce_scatter_direct_kernel(
    Peers peers, int rank, int nranks, const T* const* __restrict__ sends, T* __restrict__ out, int64_t outer,
    int64_t inner, int64_t extent, const int64_t* __restrict__ sizes, const int64_t* __restrict__ offs) {
  hap::pdl_wait();
  SignalPage* sig = reinterpret_cast<SignalPage*>(peers.base[rank]);
  const uint64_t epoch = *reinterpret_cast<volatile uint64_t*>(&sig->epoch);
  const bool peer_thread = threadIdx.x < nranks && threadIdx.x != rank;
  if (blockIdx.x == 0 && peer_thread)
    st_release_sys(&reinterpret_cast<SignalPage*>(peers.base[threadIdx.x])->ready[rank], epoch + 1);
  if (peer_thread)
    if (!peers.nosync) while (ld_acquire_sys(&sig->ready[threadIdx.x]) < epoch + 1) __nanosleep(64);
  __syncthreads();
  const int64_t rows = sizes[rank], off = offs[rank];
  const int64_t per = rows * inner, total = outer * per;
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  constexpr int kv = 16 / sizeof(T);
  bool vec = inner % kv == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  for (int p = 0; p < nranks; ++p) vec = vec && (reinterpret_cast<uintptr_t>(sends[p]) & 15) == 0;
  if (vec) {
    const int64_t per4 = per / kv, total4 = outer * per4;
    for (int64_t e = tid; e < total4; e += stride) {
      const int64_t o = e / per4, rem = e - o * per4;
      const int64_t at = (o * extent + off) * inner / kv + rem;   // int4 index in a partial
      int4 v[kMaxRanks];   // every rank's load in flight before the sum (registers: fully unrolled)
#pragma unroll
      for (int q = 0; q < kMaxRanks; ++q)
        if (q < nranks) v[q] = reinterpret_cast<const int4*>(sends[q])[at];
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int q = 0; q < kMaxRanks; ++q)
        if (q < nranks) add8<T>(acc, v[q]);
      int4 r;
      if constexpr (sizeof(T) == 2) {
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
      } else {
        float* f = reinterpret_cast<float*>(&r);
#pragma unroll
        for (int i = 0; i < 4; ++i) f[i] = acc[i];
      }
      reinterpret_cast<int4*>(out)[e] = r;
    }
  } else {
    for (int64_t e = tid; e < total; e += stride) {
      const int64_t o = e / per, rem = e - o * per;
      const int64_t at = (o * extent + off) * inner + rem;
      float acc = 0.f;
      for (int q = 0; q < nranks; ++q) acc += to_f32(sends[q][at]);
      out[e] = from_f32<T>(acc);
    }
  }
  if (grid_barrier(sig) && threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      st_release_sys(&reinterpret_cast<SignalPage*>(peers.base[p])->done[rank], epoch + 1);
    }
    sig->epoch = epoch + 1;
  }
  if (peer_thread)
    if (!peers.nosync) while (ld_acquire_sys(&sig->done[threadIdx.x]) < epoch + 1) __nanosleep(64);
}


// All-reduce over registered buffers (two-shot, one kernel): the tensor is
// cut into nranks chunks of whole 8-element groups; rank c reduces chunk c
// straight out of every rank's registered input (16-byte NVLink loads, all
// in flight before the sum, fp32 accumulation in rank order 0..m-1, one
// rounding — the LocalGroup sum bit for bit) and stores the result into
// every rank's registered output.  Each element is read and then written by
// the same thread, so in == out (in-place gradient buckets) is safe.
// Protocol (epoch e): armed[r] = e+1 on every peer at start (my input is
// complete and my output no longer read by earlier work on my stream), wait
// for every peer's armed; reduce + push; grid barrier; done[r] = e+1 on every
// peer; wait for every peer's done (my output complete, my input released).
template <typename T>
__global__ void __launch_bounds__(kThreads) p2p_all_reduce_kernel(Peers peers, int rank, int nranks,
                                                                  const T* const* __restrict__ ins,
                                                                  T* const* __restrict__ outs, int64_t count) {
  hap::pdl_wait();
  SignalPage* sig = reinterpret_cast<SignalPage*>(peers.base[rank]);
  const uint64_t epoch = *reinterpret_cast<volatile uint64_t*>(&sig->epoch);
  const bool peer_thread = threadIdx.x < nranks && threadIdx.x != rank;
  if (blockIdx.x == 0 && peer_thread)
    st_release_sys(&reinterpret_cast<SignalPage*>(peers.base[threadIdx.x])->armed[rank], epoch + 1);
  if (peer_thread)
    if (!peers.nosync) while (ld_acquire_sys(&sig->armed[threadIdx.x]) < epoch + 1) __nanosleep(64);
  __syncthreads();
  constexpr int kv = 16 / sizeof(T);
  const int64_t groups = count / 8;                     // whole 8-element groups, split into chunks
  const int64_t g0 = groups * rank / nranks, g1 = groups * (rank + 1) / nranks;
  const int64_t lo = g0 * 8, hi = rank == nranks - 1 ? count : g1 * 8;   // the tail goes to the last rank
  const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  bool vec = true;
  for (int p = 0; p < nranks; ++p)
    vec = vec && ((reinterpret_cast<uintptr_t>(ins[p]) | reinterpret_cast<uintptr_t>(outs[p])) & 15) == 0;
  int64_t scalar_from = lo;
  if (vec) {
    const int64_t n4 = (g1 * 8 - lo) / kv;
    for (int64_t e = tid; e < n4; e += stride) {
      const int64_t at = lo / kv + e;
      int4 v[kMaxRanks];
#pragma unroll
      for (int q = 0; q < kMaxRanks; ++q)
        if (q < nranks) v[q] = reinterpret_cast<const int4*>(ins[q])[at];
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int q = 0; q < kMaxRanks; ++q)
        if (q < nranks) add8<T>(acc, v[q]);
      int4 r;
      if constexpr (sizeof(T) == 2) {
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&r);
#pragma unroll
        for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
      } else {
        float* f = reinterpret_cast<float*>(&r);
#pragma unroll
        for (int i = 0; i < 4; ++i) f[i] = acc[i];
      }
#pragma unroll
      for (int q = 0; q < kMaxRanks; ++q)
        if (q < nranks) reinterpret_cast<int4*>(outs[(rank + q) % nranks])[at] = r;   // own output last-ish
    }
    scalar_from = g1 * 8;
  }
  for (int64_t e = scalar_from + tid; e < hi; e += stride) {
    float acc = 0.f;
    for (int q = 0; q < nranks; ++q) acc += to_f32(ins[q][e]);
    const T r = from_f32<T>(acc);
    for (int q = 0; q < nranks; ++q) outs[q][e] = r;
  }
  if (grid_barrier(sig) && threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      st_release_sys(&reinterpret_cast<SignalPage*>(peers.base[p])->done[rank], epoch + 1);
      st_release_sys(&reinterpret_cast<SignalPage*>(peers.base[p])->ready[rank], epoch + 1);
    }
    sig->epoch = epoch + 1;
  }
  if (peer_thread)
    if (!peers.nosync) while (ld_acquire_sys(&sig->done[threadIdx.x]) < epoch + 1) __nanosleep(64);
}

// All-to-all by pushing contiguous chunks: rank r stores chunk k of its send
// buffer (elements [send_off[k], send_off[k] + cnt[k])) straight into rank
// k's registered receive buffer at dst_off[k] (its rank-ordered receive
// layout), own chunk included.  Same armed / ready protocol as the push
// all-gather.
template <typename T>
__global__ void __launch_bounds__(kThreads) p2p_all_to_all_kernel(Peers peers, int rank, int nranks,
                                                                  const T* __restrict__ send,
                                                                  T* const* __restrict__ recvs,
                                                                  const int64_t* __restrict__ send_off,
                                                                  const int64_t* __restrict__ cnt,
                                                                  const int64_t* __restrict__ dst_off) {
  hap::pdl_wait();
  SignalPage* sig = reinterpret_cast<SignalPage*>(peers.base[rank]);
  const uint64_t epoch = *reinterpret_cast<volatile uint64_t*>(&sig->epoch);
  const bool peer_thread = threadIdx.x < nranks && threadIdx.x != rank;
  if (blockIdx.x == 0 && peer_thread)
    st_release_sys(&reinterpret_cast<SignalPage*>(peers.base[threadIdx.x])->armed[rank], epoch + 1);
  if (peer_thread)
    if (!peers.nosync) while (ld_acquire_sys(&sig->armed[threadIdx.x]) < epoch + 1) __nanosleep(64);
  __syncthreads();
  for (int q = 1; q <= nranks; ++q) {
    const int k = (rank + q) % nranks;   // peers staggered across ranks, own chunk last
    if (cnt[k] > 0) copy_elems(recvs[k] + dst_off[k], send + send_off[k], cnt[k]);
  }
  if (grid_barrier(sig) && threadIdx.x == 0) {
    __threadfence_system();
    for (int p = 0; p < nranks; ++p) {
      if (p == rank) continue;
      SignalPage* peer_sig = reinterpret_cast<SignalPage*>(peers.base[p]);
      st_release_sys(&peer_sig->ready[rank], epoch + 1);
      st_release_sys(&peer_sig->done[rank], epoch + 1);
    }
    sig->epoch = epoch + 1;
  }
  if (peer_thread)
    if (!peers.nosync) while (ld_acquire_sys(&sig->ready[threadIdx.x]) < epoch + 1) __nanosleep(64);
}

}  // namespace
}  // namespace hap

using namespace hap;

extern "C" hap_status hap_p2p_probe(void* ctx, int mode, int64_t chunk_bytes, int sm_cap, void* stream) {
  auto* s = static_cast<Symm*>(ctx);
  HAP_CHECK_ARG(s && mode >= 0 && mode <= 4 && chunk_bytes > 0 && chunk_bytes % 16 == 0 &&
                    chunk_bytes * s->nranks <= hap_symm_capacity(ctx),
                "hap_p2p_probe: bad arguments");
  Peers peers{};
  peers.nosync = p2p_nosync();
  for (int p = 0; p < s->nranks; ++p) peers.base[p] = s->peers[p];
  const int grid = capped_grid(static_cast<int64_t>(sm_count()), sm_cap);
  launch_k(p2p_probe_kernel, dim3(grid), dim3(kThreads), 0, static_cast<cudaStream_t>(stream), peers, s->rank,
           s->nranks, mode, chunk_bytes);
  return launch_status("p2p probe");
}

extern "C" hap_status hap_symm_create(void** out, int64_t bytes, int rank, int nranks) {
  HAP_CHECK_ARG(out && bytes > 0 && nranks >= 1 && nranks <= kMaxRanks && rank >= 0 && rank < nranks,
                "hap_symm_create: bad arguments");
  auto* s = new Symm();
  s->rank = rank;
  s->nranks = nranks;
  s->bytes = kSignalBytes + static_cast<size_t>(bytes);
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(&s->local), s->bytes);
  if (e != cudaSuccess) {
    delete s;
    set_error(std::string("hap_symm_create: cudaMalloc: ") + cudaGetErrorString(e));
    return HAP_ERR_CUDA;
  }
  // The signal page must be zero before any peer can see this arena and
  // before this rank's first peer kernel: a plain cudaMemset runs on the
  // legacy stream, which does not order against the executor's non-blocking
  // streams, so a fresh process's first collective could read a stale epoch
  // or have its peers' first flags wiped — both ranks then wait inside the
  // same collective forever (tests/multi/peer_ranks.py, first run of a
  // process).  Zero it on a private stream and wait for it here.
  cudaStream_t st = nullptr;
  HAP_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  e = cudaMemsetAsync(s->local, 0, kSignalBytes, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (e != cudaSuccess) {
    cudaFree(s->local);
    delete s;
    set_error(std::string("hap_symm_create: zeroing the signal page: ") + cudaGetErrorString(e));
    return HAP_ERR_CUDA;
  }
  s->peers[rank] = s->local;
  *out = s;
  return HAP_OK;
}

extern "C" hap_status hap_symm_handle(void* ctx, uint8_t* out64) {
  auto* s = static_cast<Symm*>(ctx);
  HAP_CHECK_ARG(s && out64, "hap_symm_handle: bad arguments");
  cudaIpcMemHandle_t h;
  HAP_CUDA_TRY(cudaIpcGetMemHandle(&h, s->local));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  std::memcpy(out64, &h, 64);
  return HAP_OK;
}

extern "C" hap_status hap_symm_open(void* ctx, const uint8_t* handles) {
  auto* s = static_cast<Symm*>(ctx);
  HAP_CHECK_ARG(s && handles, "hap_symm_open: bad arguments");
  for (int p = 0; p < s->nranks; ++p) {
    if (p == s->rank) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handles + 64 * p, 64);
    void* ptr = nullptr;
    HAP_CUDA_TRY(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
    s->peers[p] = static_cast<char*>(ptr);
  }
  return HAP_OK;
}

extern "C" hap_status hap_symm_destroy(void* ctx) {
  auto* s = static_cast<Symm*>(ctx);
  if (!s) return HAP_OK;
  for (auto& kv : s->opened) cudaIpcCloseMemHandle(kv.second);
  if (!s->local_open)
    for (int p = 0; p < s->nranks; ++p)
      if (p != s->rank && s->peers[p]) cudaIpcCloseMemHandle(s->peers[p]);
  cudaFree(s->local);
  delete s;
  return HAP_OK;
}

namespace {
// Base of the allocation holding `ptr` (driver cuMemGetAddressRange).
bool alloc_base(const void* ptr, char** base) {
  ensure_context();
  using Fn = int (*)(uint64_t*, size_t*, uint64_t);
  static Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<Fn>(p);
  });
  uint64_t b = 0;
  size_t sz = 0;
  if (!fn || fn(&b, &sz, reinterpret_cast<uint64_t>(ptr)) != 0) return false;
  *base = reinterpret_cast<char*>(b);
  return true;
}
}  // namespace

extern "C" hap_status hap_p2p_buffer_handle(void* ctx, const void* buf, uint8_t* out64, int64_t* base_addr,
                                            int64_t* offset) {
  auto* s = static_cast<Symm*>(ctx);
  HAP_CHECK_ARG(s && buf && out64 && base_addr && offset, "hap_p2p_buffer_handle: bad arguments");
  char* base = nullptr;
  HAP_CHECK_ARG(alloc_base(buf, &base), "hap_p2p_buffer_handle: not a device allocation");
  cudaIpcMemHandle_t h;
  HAP_CUDA_TRY(cudaIpcGetMemHandle(&h, base));
  std::memcpy(out64, &h, 64);
  *base_addr = static_cast<int64_t>(reinterpret_cast<uintptr_t>(base));
  *offset = static_cast<const char*>(buf) - base;
  return HAP_OK;
}

extern "C" hap_status hap_p2p_buffer_open(void* ctx, const void* own, const uint8_t* handles64xn,
                                          const int64_t* base_addrs, const int64_t* offsets, void** out_ptrs) {
  auto* s = static_cast<Symm*>(ctx);
  HAP_CHECK_ARG(s && own && handles64xn && base_addrs && offsets && out_ptrs, "hap_p2p_buffer_open: bad arguments");
  for (int p = 0; p < s->nranks; ++p) {
    if (p == s->rank) {
      out_ptrs[p] = const_cast<void*>(own);
      continue;
    }
    (void)base_addrs;
    const auto key = std::make_pair(p, std::string(reinterpret_cast<const char*>(handles64xn + 64 * p), 64));
    auto it = s->opened.find(key);
    if (it == s->opened.end()) {
      cudaIpcMemHandle_t h;
      std::memcpy(&h, handles64xn + 64 * p, 64);
      void* ptr = nullptr;
      HAP_CUDA_TRY(cudaIpcOpenMemHandle(&ptr, h, cudaIpcMemLazyEnablePeerAccess));
      it = s->opened.emplace(key, static_cast<char*>(ptr)).first;
    }
    out_ptrs[p] = it->second + offsets[p];
  }
  return HAP_OK;
}

extern "C" int64_t hap_symm_capacity(void* ctx) {
  auto* s = static_cast<Symm*>(ctx);
  return s ? static_cast<int64_t>(s->bytes - kSignalBytes) : 0;
}

namespace {

// CTAs for a call moving `bytes`: each CTA keeps ~64 KB of NVLink reads in
// flight (512 threads x 8 x 16 B), so small messages use few CTAs — cheaper
// grid barriers, and SMs left to the compute stream when the call runs on a
// side stream — and large ones one CTA per (capped) SM.
inline int p2p_grid(int64_t bytes, int sm_cap) {
  const int64_t want = std::max<int64_t>(4, (bytes + 65535) / 65536);
  return capped_grid(want, sm_cap);
}

// Every CTA of a peer-memory kernel spins on flags (peers' and the grid
// barrier's), so the whole grid must become resident.  Plain launches (the
// default): the grid is small (p2p_grid, and the executor caps side-stream and
// in-process peer kernels at 32 / 16 CTAs), and the only other kernels on the
// GPU are finite (GEMMs, elementwise), so the missing CTAs become resident as
// those finish.  HAP_P2P_COOP=1 launches cooperatively instead, which
// guarantees co-residency up front — but measured on B200, a running
// cooperative kernel keeps kernels of OTHER streams from being scheduled: two
// in-process ranks deadlocked with rank 0's plain elementwise kernel queued
// behind rank 1's spinning cooperative all-reduce (tests/multi/peer_ranks.py),
// and in one process per GPU it would stall the compute stream while a
// side-stream collective waits for its peers.
int p2p_cooperative() {
  static int on = [] {
    const char* v = getenv("HAP_P2P_COOP");
    return v ? atoi(v) : 0;
  }();
  return on;
}

template <typename... KArgs, typename... Args>
void launch_p2p(void (*kern)(KArgs...), int grid, cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  attr[1].id = cudaLaunchAttributeCooperative;
  attr[1].val.cooperative = p2p_cooperative();
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <typename T>
hap_status p2p_launch(void (*kern)(Peers, int, int, const T*, T*, int64_t, int64_t, int64_t, const int64_t*,
                                   const int64_t*),
                      Symm* s, const void* send, void* out, int64_t outer, int64_t inner, int64_t extent,
                      const int64_t* dev_sizes, const int64_t* dev_offs, int64_t bytes, int sm_cap,
                      cudaStream_t stream) {
  Peers peers{};
  peers.nosync = p2p_nosync();
  for (int p = 0; p < s->nranks; ++p) peers.base[p] = s->peers[p];
  const int grid = p2p_grid(bytes, sm_cap);   // every CTA resident (they spin on peer flags)
  launch_p2p(kern, grid, stream, peers, s->rank, s->nranks, static_cast<const T*>(send), static_cast<T*>(out), outer,
             inner, extent, dev_sizes, dev_offs);
  return launch_status("p2p kernel");
}

}  // namespace

extern "C" hap_status hap_p2p_all_gather_v(void* ctx, const void* send, void* recv, hap_dtype dtype,
                                           int64_t outer, int64_t inner, int64_t extent,
                                           const int64_t* dev_sizes, const int64_t* dev_offsets,
                                           int64_t max_chunk_elems, int sm_cap, void* stream) {
  auto* s = static_cast<Symm*>(ctx);
  HAP_CHECK_ARG(s && dev_sizes && dev_offsets, "hap_p2p_all_gather_v: bad arguments");
  HAP_CHECK_ARG(max_chunk_elems * static_cast<int64_t>(dtype_size(dtype)) <= hap_symm_capacity(ctx),
                "hap_p2p_all_gather_v: shard larger than the symmetric staging buffer");
  auto st = static_cast<cudaStream_t>(stream);
  const int64_t bytes = max_chunk_elems * s->nranks * static_cast<int64_t>(dtype_size(dtype));
  if (dtype == HAP_BF16)
    return p2p_launch<__nv_bfloat16>(p2p_all_gather_kernel<__nv_bfloat16>, s, send, recv, outer, inner, extent,
                                     dev_sizes, dev_offsets, bytes, sm_cap, st);
  return p2p_launch<float>(p2p_all_gather_kernel<float>, s, send, recv, outer, inner, extent, dev_sizes, dev_offsets,
                           bytes, sm_cap, st);
}

extern "C" hap_status hap_p2p_all_gather_push(void* ctx, const void* send, void* const* dev_outs, hap_dtype dtype,
                                              int64_t outer, int64_t inner, int64_t extent, const int64_t* dev_sizes,
                                              const int64_t* dev_offsets, int64_t total_elems, int sm_cap,
                                              void* stream) {
  auto* s = static_cast<Symm*>(ctx);
  HAP_CHECK_ARG(s && dev_outs && dev_sizes && dev_offsets, "hap_p2p_all_gather_push: bad arguments");
  Peers peers{};
  peers.nosync = p2p_nosync();
  for (int p = 0; p < s->nranks; ++p) peers.base[p] = s->peers[p];
  // every CTA spins on peer flags: all resident, one per (capped) SM at most
  const int grid = p2p_grid(total_elems * static_cast<int64_t>(dtype_size(dtype)), sm_cap);
  auto st = static_cast<cudaStream_t>(stream);
  if (dtype == HAP_BF16)
    launch_p2p(p2p_all_gather_push_kernel<__nv_bfloat16>, grid, st, peers, s->rank, s->nranks, static_cast<const __nv_bfloat16*>(send), reinterpret_cast<__nv_bfloat16* const*>(dev_outs),
             outer, inner, extent, dev_sizes, dev_offsets);
  else
    launch_p2p(p2p_all_gather_push_kernel<float>, grid, st, peers, s->rank, s->nranks,
             static_cast<const float*>(send), reinterpret_cast<float* const*>(dev_outs), outer, inner, extent,
             dev_sizes, dev_offsets);
  return launch_status("p2p push all-gather");
}

extern "C" hap_status hap_p2p_reduce_scatter_direct(void* ctx, const void* const* dev_sends, void* recv,
                                                    hap_dtype dtype, int64_t outer, int64_t inner, int64_t extent,
                                                    const int64_t* dev_sizes, const int64_t* dev_offsets,
                                                    int64_t recv_elems, int sm_cap, void* stream) {
  auto* s = static_cast<Symm*>(ctx);
  HAP_CHECK_ARG(s && dev_sends && recv && dev_sizes && dev_offsets, "hap_p2p_reduce_scatter_direct: bad arguments");
  Peers peers{};
  peers.nosync = p2p_nosync();
  for (int p = 0; p < s->nranks; ++p) peers.base[p] = s->peers[p];
  const int grid = p2p_grid(recv_elems * s->nranks * static_cast<int64_t>(dtype_size(dtype)), sm_cap);
  auto st = static_cast<cudaStream_t>(stream);
  if (dtype == HAP_BF16)
    launch_p2p(p2p_reduce_scatter_direct_kernel<__nv_bfloat16>, grid, st, peers, s->rank, s->nranks, reinterpret_cast<const __nv_bfloat16* const*>(dev_sends), static_cast<__nv_bfloat16*>(recv),
             outer, inner, extent, dev_sizes, dev_offsets);
  else
    launch_p2p(p2p_reduce_scatter_direct_kernel<float>, grid, st, peers, s->rank, s->nranks,
             reinterpret_cast<const float* const*>(dev_sends), static_cast<float*>(recv), outer, inner, extent,
             dev_sizes, dev_offsets);
  return launch_status("p2p direct reduce-scatter");
}

extern "C" hap_status hap_p2p_reduce_scatter_v(void* ctx, const void* send, void* recv, hap_dtype dtype,
                                               int64_t outer, int64_t inner, int64_t extent,
                                               const int64_t* dev_sizes, const int64_t* dev_offsets,
                                               int sm_cap, void* stream) {
  auto* s = static_cast<Symm*>(ctx);
  HAP_CHECK_ARG(s && dev_sizes && dev_offsets, "hap_p2p_reduce_scatter_v: bad arguments");
  HAP_CHECK_ARG(outer * extent * inner * static_cast<int64_t>(dtype_size(dtype)) <= hap_symm_capacity(ctx),
                "hap_p2p_reduce_scatter_v: tensor larger than the symmetric staging buffer");
  auto st = static_cast<cudaStream_t>(stream);
  const int64_t bytes = outer * extent * inner * static_cast<int64_t>(dtype_size(dtype));
  if (dtype == HAP_BF16)
    return p2p_launch<__nv_bfloat16>(p2p_reduce_scatter_kernel<__nv_bfloat16>, s, send, recv, outer, inner, extent,
                                     dev_sizes, dev_offsets, bytes, sm_cap, st);
  return p2p_launch<float>(p2p_reduce_scatter_kernel<float>, s, send, recv, outer, inner, extent, dev_sizes,
                           dev_offsets, bytes, sm_cap, st);
}

extern "C" hap_status hap_symm_open_local(void* ctx, const int64_t* peer_bases) {
  auto* s = static_cast<Symm*>(ctx);
  HAP_CHECK_ARG(s && peer_bases, "hap_symm_open_local: bad arguments");
  for (int p = 0; p < s->nranks; ++p) {
    HAP_CHECK_ARG(peer_bases[p] != 0, "hap_symm_open_local: null peer arena");
    s->peers[p] = reinterpret_cast<char*>(static_cast<uintptr_t>(peer_bases[p]));
  }
  HAP_CHECK_ARG(s->peers[s->rank] == s->local, "hap_symm_open_local: own entry is not this context's arena");
  s->local_open = true;
  return HAP_OK;
}

extern "C" hap_status hap_symm_peek(void* ctx, void* host512) {
  auto* s = static_cast<Symm*>(ctx);
  HAP_CHECK_ARG(s && host512, "hap_symm_peek: bad arguments");
  cudaStream_t st = nullptr;
  HAP_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  cudaError_t e = cudaMemcpyAsync(host512, s->local, kSignalBytes, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (e != cudaSuccess) {
    set_error(std::string("hap_symm_peek: ") + cudaGetErrorString(e));
    return HAP_ERR_CUDA;
  }
  return HAP_OK;
}

extern "C" void* hap_symm_local_base(void* ctx) {
  auto* s = static_cast<Symm*>(ctx);
  return s ? s->local : nullptr;
}

extern "C" hap_status hap_p2p_all_reduce(void* ctx, const void* const* dev_ins, void* const* dev_outs, hap_dtype dtype,
                                         int64_t count, int sm_cap, void* stream) {
  auto* s = static_cast<Symm*>(ctx);
  HAP_CHECK_ARG(s && dev_ins && dev_outs && count >= 0, "hap_p2p_all_reduce: bad arguments");
  Peers peers{};
  peers.nosync = p2p_nosync();
  for (int p = 0; p < s->nranks; ++p) peers.base[p] = s->peers[p];
  // bytes this rank moves: its chunk from every peer and to every peer
  const int grid = p2p_grid(2 * count * static_cast<int64_t>(dtype_size(dtype)), sm_cap);
  auto st = static_cast<cudaStream_t>(stream);
  if (dtype == HAP_BF16)
    launch_p2p(p2p_all_reduce_kernel<__nv_bfloat16>, grid, st, peers, s->rank, s->nranks,
               reinterpret_cast<const __nv_bfloat16* const*>(dev_ins), reinterpret_cast<__nv_bfloat16* const*>(dev_outs),
               count);
  else
    launch_p2p(p2p_all_reduce_kernel<float>, grid, st, peers, s->rank, s->nranks,
               reinterpret_cast<const float* const*>(dev_ins), reinterpret_cast<float* const*>(dev_outs), count);
  return launch_status("p2p all-reduce");
}

extern "C" hap_status hap_p2p_all_to_all(void* ctx, const void* send, void* const* dev_recvs, hap_dtype dtype,
                                         const int64_t* dev_send_off, const int64_t* dev_counts,
                                         const int64_t* dev_dst_off, int64_t max_elems, int sm_cap, void* stream) {
  auto* s = static_cast<Symm*>(ctx);
  HAP_CHECK_ARG(s && dev_recvs && dev_send_off && dev_counts && dev_dst_off, "hap_p2p_all_to_all: bad arguments");
  Peers peers{};
  peers.nosync = p2p_nosync();
  for (int p = 0; p < s->nranks; ++p) peers.base[p] = s->peers[p];
  const int grid = p2p_grid(max_elems * static_cast<int64_t>(dtype_size(dtype)), sm_cap);
  auto st = static_cast<cudaStream_t>(stream);
  if (dtype == HAP_BF16)
    launch_p2p(p2p_all_to_all_kernel<__nv_bfloat16>, grid, st, peers, s->rank, s->nranks,
               static_cast<const __nv_bfloat16*>(send), reinterpret_cast<__nv_bfloat16* const*>(dev_recvs), dev_send_off,
               dev_counts, dev_dst_off);
  else
    launch_p2p(p2p_all_to_all_kernel<float>, grid, st, peers, s->rank, s->nranks, static_cast<const float*>(send),
               reinterpret_cast<float* const*>(dev_recvs), dev_send_off, dev_counts, dev_dst_off);
  return launch_status("p2p all-to-all");
}
