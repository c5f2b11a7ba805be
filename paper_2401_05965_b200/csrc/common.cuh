// Shared helpers for the HAP B200 executor kernels (sm_100a only).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "../../include/hap_b200.h"

namespace hap {

// Last error message (thread-local) surfaced through hap_last_error().
void set_error(const std::string& msg);

#define HAP_CUDA_TRY(expr)                                                       \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::hap::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));      \
      return HAP_ERR_CUDA;                                                       \
    }                                                                            \
  } while (0)

#define HAP_CHECK_ARG(cond, msg)                                                 \
  do {                                                                           \
    if (!(cond)) {                                                               \
      ::hap::set_error(msg);                                                     \
      return HAP_ERR_ARG;                                                        \
    }                                                                            \
  } while (0)

inline hap_status launch_status(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return HAP_ERR_CUDA;
  }
  return HAP_OK;
}

// SM count of the current device (cached per device).
int sm_count();

// Make the current device's primary context current in the calling thread
// (once per thread) before a driver-API call such as cuTensorMapEncodeTiled:
// a thread whose first CUDA call is into this library (ranks stepped from
// worker threads) would otherwise have no context and the call would fail.
void ensure_context();

// Per-stream device scratch for kernels that need a workspace (ordered
// reduction partials, split-K partial tiles, arrival counters).  Launches on
// one stream are ordered, so they share a slot.  A slot grows only outside
// stream capture (returns false during capture when too small); a buffer it
// outgrows is retired, never freed, because a CUDA graph captured earlier may
// still hold its address.  `zeroed` slots are cleared on allocation: kernels
// that use them as counters leave them at zero when they finish.
enum ScratchSlot { kScratchSplitWs = 0, kScratchReduce, kScratchReduceTickets,
                   kScratchStreamK, kScratchStreamKFlags, kScratchSlots };
bool stream_scratch(cudaStream_t stream, int slot, size_t bytes, bool zeroed, void** out);

// Grid size for a capped, persistent launch: at most `sm_cap` CTAs (one per
// SM when each CTA is sized to fill an SM), never more than `work_blocks`.
inline int capped_grid(int64_t work_blocks, int sm_cap) {
  int cap = sm_cap > 0 ? sm_cap : sm_count();
  if (cap > sm_count()) cap = sm_count();
  int64_t g = work_blocks < cap ? work_blocks : cap;
  return g < 1 ? 1 : static_cast<int>(g);
}

// Programmatic dependent launch (PDL): every kernel is launched with
// programmatic stream serialisation, so the next kernel in the stream (or
// CUDA graph) is scheduled while this one drains; each kernel first waits for
// its predecessor's memory (griddepcontrol.wait) and then immediately lets its
// own successor start launching.  Setup that touches no global memory (smem
// barriers, TMEM allocation, descriptor prefetch) runs before the wait and so
// overlaps the previous kernel's tail.  Enabled with HAP_PDL=1 (default off:
// measured slower on the mixed GEMM/elementwise step, faster GEMM-to-GEMM).
int pdl_enabled();

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
// Short grid-stride kernels only wait: their successors launch at their
// completion (an early trigger let the next GEMM's CTAs occupy SMs while the
// elementwise kernel still streamed, which measured slower end to end).
__device__ __forceinline__ void pdl_enter() { pdl_wait(); }

int carveout_pref();

// HAP_CARVEOUT=<percent>: every kernel asks for that shared-memory carveout,
// so consecutive GEMM (225 KB smem) and elementwise launches need not
// re-partition L1/shared memory between kernels.  Default: the driver's
// choice (forcing 100 % measured slower).
template <typename K>
inline void set_carveout(K kern) {
  // per launch (a static flag here would be shared by every kernel of the
  // same signature); the default -1 sets nothing
  const int pref = carveout_pref();
  if (pref >= 0) cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pref);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                            Args&&... args) {
  set_carveout(kern);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

__device__ __forceinline__ float to_f32(float v) { return v; }
__device__ __forceinline__ float to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// Round a pair of fp32 values to storage precision T and back (in place):
// for bf16 one F2FP pack + two shifts on the ALU pipe — the same
// round-to-nearest-even as from_f32 per value (F2F, a quarter-rate XU op that
// MUFU shares) — so vectorised kernels round two values per instruction.
template <typename T> __device__ __forceinline__ void round2(float& a, float& b);
template <> __device__ __forceinline__ void round2<float>(float&, float&) {}
template <> __device__ __forceinline__ void round2<__nv_bfloat16>(float& a, float& b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  const uint32_t u = *reinterpret_cast<const uint32_t*>(&h);
  a = __uint_as_float(u << 16);
  b = __uint_as_float(u & 0xffff0000u);
}

// Elementwise unary functions (interpreter.py:141-143), shared by the
// elementwise kernels and the GEMM's fused epilogues so both round alike.
__device__ __forceinline__ float unary_fwd(int tag, float x) {
  switch (tag) {
    case HAP_EXP: return __expf(x);
    case HAP_NEG: return -x;
    case HAP_RELU: return fmaxf(x, 0.f);
    case HAP_SIGMOID: {   // two MUFU ops: 2^(-x log2 e), then 1 / (1 + that) (~2 ulp fp32)
      float e, y;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(x * -1.4426950408889634f));
      asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(1.f + e));
      return y;
    }
    default: return tanhf(x);
  }
}

template <int TAG>
__device__ __forceinline__ float unary_fwd_t(float x) { return unary_fwd(TAG, x); }

// d/dx f at x, given y = f(x).
__device__ __forceinline__ float unary_deriv(int tag, float x, float y) {
  switch (tag) {
    case HAP_EXP: return y;
    case HAP_NEG: return -1.f;
    case HAP_RELU: return x > 0.f ? 1.f : 0.f;
    case HAP_SIGMOID: return y * (1.f - y);
    default: return 1.f - y * y;
  }
}

inline size_t dtype_size(hap_dtype t) { return t == HAP_BF16 ? 2 : 4; }

}  // namespace hap

// Dispatch a (input dtype, output dtype) pair to a templated body.
#define HAP_DISPATCH_IO(IN, OUT, ...)                                            \
  [&]() -> hap_status {                                                          \
    if ((IN) == HAP_BF16 && (OUT) == HAP_BF16) {                                 \
      using Tin = __nv_bfloat16; using Tout = __nv_bfloat16; return __VA_ARGS__(); \
    } else if ((IN) == HAP_BF16 && (OUT) == HAP_F32) {                           \
      using Tin = __nv_bfloat16; using Tout = float; return __VA_ARGS__();       \
    } else if ((IN) == HAP_F32 && (OUT) == HAP_BF16) {                           \
      using Tin = float; using Tout = __nv_bfloat16; return __VA_ARGS__();       \
    } else {                                                                     \
      using Tin = float; using Tout = float; return __VA_ARGS__();               \
    }                                                                            \
  }()
