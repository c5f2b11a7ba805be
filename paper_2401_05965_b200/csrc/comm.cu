// Collectives of the distributed program over NCCL (NVLink 5 / NVSwitch).
//
// The reference simulates them with numpy (interpreter.py:69-101); here each
// process owns one device and the uneven, ratio-weighted shard sizes of the
// plan's shard table become per-rank element counts.  Two gather
// implementations mirror the two collective kinds the planner prices
// (cost_model.py:203-219): `all_gather` pads every chunk to the largest shard
// and runs one ring all-gather; `grouped_broadcast` issues one broadcast per
// shard at its true size.  Reduce-scatter uses the padded layout the cost
// model charges; all-to-all is grouped point-to-point.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace hap {
namespace {

struct Comm {
  ncclComm_t nccl = nullptr;
  int rank = 0;
  int nranks = 1;
};

#define HAP_NCCL_TRY(expr)                                                     \
  do {                                                                         \
    ncclResult_t _r = (expr);                                                  \
    if (_r != ncclSuccess) {                                                   \
      ::hap::set_error(std::string(#expr) + ": " + ncclGetErrorString(_r));    \
      return HAP_ERR_NCCL;                                                     \
    }                                                                          \
  } while (0)

ncclDataType_t nccl_type(hap_dtype t) { return t == HAP_BF16 ? ncclBfloat16 : ncclFloat32; }

std::vector<int64_t> offsets(const int64_t* counts, int n) {
  std::vector<int64_t> off(n + 1, 0);
  for (int j = 0; j < n; ++j) off[j + 1] = off[j] + counts[j];
  return off;
}

}  // namespace
}  // namespace hap

using namespace hap;

extern "C" int hap_nccl_version(void) {
  int v = 0;
  ncclGetVersion(&v);
  return v;
}

extern "C" hap_status hap_comm_unique_id(uint8_t* out) {
  HAP_CHECK_ARG(out != nullptr, "hap_comm_unique_id: null output");
  ncclUniqueId id;
  HAP_NCCL_TRY(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, sizeof(id));
  return HAP_OK;
}

extern "C" hap_status hap_comm_init(void** out, const uint8_t* id128, int nranks, int rank) {
  HAP_CHECK_ARG(out && id128 && nranks >= 1 && rank >= 0 && rank < nranks,
                "hap_comm_init: bad arguments");
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  auto* c = new Comm();
  c->rank = rank;
  c->nranks = nranks;
  ncclResult_t r = ncclCommInitRank(&c->nccl, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    set_error(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    return HAP_ERR_NCCL;
  }
  *out = c;
  return HAP_OK;
}

extern "C" hap_status hap_comm_destroy(void* comm) {
  auto* c = static_cast<Comm*>(comm);
  if (!c) return HAP_OK;
  ncclResult_t r = ncclCommDestroy(c->nccl);
  delete c;
  if (r != ncclSuccess) {
    set_error(std::string("ncclCommDestroy: ") + ncclGetErrorString(r));
    return HAP_ERR_NCCL;
  }
  return HAP_OK;
}

extern "C" hap_status hap_all_reduce(void* comm, const void* send, void* recv, int64_t count,
                                     hap_dtype dtype, void* stream) {
  auto* c = static_cast<Comm*>(comm);
  HAP_CHECK_ARG(c != nullptr, "hap_all_reduce: null communicator");
  if (count <= 0) return HAP_OK;
  HAP_NCCL_TRY(ncclAllReduce(send, recv, count, nccl_type(dtype), ncclSum, c->nccl,
                             static_cast<cudaStream_t>(stream)));
  return HAP_OK;
}

extern "C" hap_status hap_all_gather_v(void* comm, const void* send, void* recv,
                                       const int64_t* counts, hap_dtype dtype, int padded,
                                       void* scratch, void* stream_) {
  auto* c = static_cast<Comm*>(comm);
  HAP_CHECK_ARG(c && counts, "hap_all_gather_v: bad arguments");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int n = c->nranks, me = c->rank;
  const size_t es = dtype_size(dtype);
  const auto off = offsets(counts, n);
  if (off[n] == 0) return HAP_OK;
  char* out = static_cast<char*>(recv);
  if (padded) {
    const int64_t maxc = *std::max_element(counts, counts + n);
    HAP_CHECK_ARG(scratch != nullptr, "hap_all_gather_v: padded gather needs scratch");
    char* buf = static_cast<char*>(scratch);
    if (counts[me] > 0)
      HAP_CUDA_TRY(cudaMemcpyAsync(buf + me * maxc * es, send, counts[me] * es,
                                   cudaMemcpyDeviceToDevice, stream));
    HAP_NCCL_TRY(ncclAllGather(buf + me * maxc * es, buf, maxc, nccl_type(dtype), c->nccl, stream));
    for (int j = 0; j < n; ++j)
      if (counts[j] > 0)
        HAP_CUDA_TRY(cudaMemcpyAsync(out + off[j] * es, buf + j * maxc * es, counts[j] * es,
                                     cudaMemcpyDeviceToDevice, stream));
    return HAP_OK;
  }
  if (counts[me] > 0 && send != out + off[me] * es)
    HAP_CUDA_TRY(cudaMemcpyAsync(out + off[me] * es, send, counts[me] * es,
                                 cudaMemcpyDeviceToDevice, stream));
  HAP_NCCL_TRY(ncclGroupStart());
  for (int j = 0; j < n; ++j) {
    if (j == me) continue;
    if (counts[me] > 0) HAP_NCCL_TRY(ncclSend(send, counts[me], nccl_type(dtype), j, c->nccl, stream));
    if (counts[j] > 0)
      HAP_NCCL_TRY(ncclRecv(out + off[j] * es, counts[j], nccl_type(dtype), j, c->nccl, stream));
  }
  HAP_NCCL_TRY(ncclGroupEnd());
  return HAP_OK;
}

extern "C" hap_status hap_grouped_broadcast(void* comm, const void* send, void* recv,
                                            const int64_t* counts, hap_dtype dtype, void* stream_) {
  auto* c = static_cast<Comm*>(comm);
  HAP_CHECK_ARG(c && counts, "hap_grouped_broadcast: bad arguments");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int n = c->nranks, me = c->rank;
  const size_t es = dtype_size(dtype);
  const auto off = offsets(counts, n);
  char* out = static_cast<char*>(recv);
  HAP_NCCL_TRY(ncclGroupStart());
  for (int j = 0; j < n; ++j) {
    if (counts[j] == 0) continue;
    const void* src = j == me ? send : out + off[j] * es;
    HAP_NCCL_TRY(ncclBroadcast(src, out + off[j] * es, counts[j], nccl_type(dtype), j, c->nccl, stream));
  }
  HAP_NCCL_TRY(ncclGroupEnd());
  return HAP_OK;
}

extern "C" hap_status hap_reduce_scatter_v(void* comm, const void* send, void* recv,
                                           const int64_t* counts, hap_dtype dtype, void* scratch,
                                           void* stream_) {
  auto* c = static_cast<Comm*>(comm);
  HAP_CHECK_ARG(c && counts && scratch, "hap_reduce_scatter_v: bad arguments");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int n = c->nranks, me = c->rank;
  const size_t es = dtype_size(dtype);
  const auto off = offsets(counts, n);
  const int64_t maxc = *std::max_element(counts, counts + n);
  if (maxc == 0) return HAP_OK;
  char* buf = static_cast<char*>(scratch);
  const char* in = static_cast<const char*>(send);
  for (int j = 0; j < n; ++j)
    if (counts[j] > 0)
      HAP_CUDA_TRY(cudaMemcpyAsync(buf + j * maxc * es, in + off[j] * es, counts[j] * es,
                                   cudaMemcpyDeviceToDevice, stream));
  HAP_NCCL_TRY(ncclReduceScatter(buf, buf + me * maxc * es, maxc, nccl_type(dtype), ncclSum,
                                 c->nccl, stream));
  if (counts[me] > 0)
    HAP_CUDA_TRY(cudaMemcpyAsync(recv, buf + me * maxc * es, counts[me] * es,
                                 cudaMemcpyDeviceToDevice, stream));
  return HAP_OK;
}

extern "C" hap_status hap_all_to_all_v(void* comm, const void* send, const int64_t* send_counts,
                                       void* recv, const int64_t* recv_counts, hap_dtype dtype,
                                       void* stream_) {
  auto* c = static_cast<Comm*>(comm);
  HAP_CHECK_ARG(c && send_counts && recv_counts, "hap_all_to_all_v: bad arguments");
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  const int n = c->nranks, me = c->rank;
  const size_t es = dtype_size(dtype);
  const auto soff = offsets(send_counts, n), roff = offsets(recv_counts, n);
  const char* in = static_cast<const char*>(send);
  char* out = static_cast<char*>(recv);
  if (send_counts[me] > 0)
    HAP_CUDA_TRY(cudaMemcpyAsync(out + roff[me] * es, in + soff[me] * es, send_counts[me] * es,
                                 cudaMemcpyDeviceToDevice, stream));
  HAP_NCCL_TRY(ncclGroupStart());
  for (int j = 0; j < n; ++j) {
    if (j == me) continue;
    if (send_counts[j] > 0)
      HAP_NCCL_TRY(ncclSend(in + soff[j] * es, send_counts[j], nccl_type(dtype), j, c->nccl, stream));
    if (recv_counts[j] > 0)
      HAP_NCCL_TRY(ncclRecv(out + roff[j] * es, recv_counts[j], nccl_type(dtype), j, c->nccl, stream));
  }
  HAP_NCCL_TRY(ncclGroupEnd());
  return HAP_OK;
}
