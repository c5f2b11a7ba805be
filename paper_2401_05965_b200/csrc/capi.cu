// Library-level entry points: error reporting, version, device queries.
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <utility>
#include <vector>

#include "common.cuh"

namespace hap {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int pdl_enabled() {
  static int on = [] {
    // Off by default: back-to-back GEMMs gain ~10% from it, but the full
    // training step measured ~2% slower with it (profiles/README.md, PDL).
    const char* v = getenv("HAP_PDL");
    return v ? atoi(v) : 0;
  }();
  return on;
}

int carveout_pref() {
  static int pref = [] {
    // default: leave the driver's choice (forcing 100 % measured slower)
    const char* v = getenv("HAP_CARVEOUT");
    return v ? atoi(v) : -1;
  }();
  return pref;
}

void ensure_context() {
  static thread_local bool done = false;
  if (done) return;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaSetDevice(dev) == cudaSuccess) done = true;
  cudaGetLastError();
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cached[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cached[dev] = n;
  }
  return cached[dev];
}

bool stream_scratch(cudaStream_t stream, int slot, size_t bytes, bool zeroed, void** out) {
  struct Entry {
    void* ptr = nullptr;
    size_t bytes = 0;
  };
  static std::mutex mu;
  static std::map<std::pair<cudaStream_t, int>, Entry> table;
  static std::vector<void*> retired;   // outgrown buffers a captured graph may reference
  if (slot < 0 || slot >= kScratchSlots) return false;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  Entry& e = table[{stream, slot * 64 + dev}];
  if (e.bytes >= bytes && e.ptr) {
    *out = e.ptr;
    return true;
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return false;
  }
  const size_t n = std::max<size_t>(std::max<size_t>(bytes, 2 * e.bytes), 1 << 16);
  void* p = nullptr;
  if (cudaMalloc(&p, n) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (zeroed && cudaMemsetAsync(p, 0, n, stream) != cudaSuccess) {   // ordered before the slot's first user
    cudaGetLastError();
    cudaFree(p);
    return false;
  }
  if (e.ptr) retired.push_back(e.ptr);
  e.ptr = p;
  e.bytes = n;
  *out = p;
  return true;
}

}  // namespace hap

extern "C" const char* hap_last_error(void) { return hap::g_last_error.c_str(); }

extern "C" int hap_abi_version(void) { return 1; }

extern "C" int hap_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return n;
}
