// Ratio-sharded GEMM for the `matmul` instruction and its adjoints.
//
// Forward   C = A . B        (reference interpreter.py:139-140, per device)
// Adjoints dA = dC . B^T,  dB = A^T . dC   (executor backward pass)
//
// tcgen05 path (bf16 in, fp32 accumulate in TMEM, bf16/fp32 out):
//   * persistent, warp-specialised CTA (256 threads, one CTA per SM):
//       warp 0  TMA producer (one elected lane)
//       warp 1  MMA issuer   (one elected lane, tcgen05.mma.cta_group::1)
//       warp 2  TMEM allocator
//       warps 4-7 epilogue   (tcgen05.ld -> registers -> global)
//   * tile 128 x BN x 64, BN in {128, 256}; smem ring of 6 / 4 stages fed by
//     TMA with 128B swizzle; double-buffered TMEM accumulator so the epilogue
//     of tile i overlaps the MMAs of tile i+1;
//   * every operand orientation the adjoints need is handled by the UMMA
//     descriptor's major-ness (K-major or MN-major) — no transposes in HBM;
//   * grid = min(tiles, sm_cap): the per-rank SM cap that emulates a slower
//     device bounds the SMs the kernel can occupy.
// SIMT path: fp32 inputs, or strides TMA cannot describe (row pitch not a
// multiple of 16 bytes) — small corpus shapes and zero-size shards.
#include <cudaTypedefs.h>

#include <cstdio>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>
#include <unordered_map>

#include "common.cuh"

namespace hap {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int UMMA_K = 16;
constexpr int kThreads = 384;   // 4 control warps + 8 epilogue warps
constexpr int kEpiWarps = 8;

// Epilogue staging: one 4 KB box (32 rows x 128 B, or two 32 x 64 B boxes)
// per epilogue warp, where the warp transposes its row-per-lane accumulator
// values into full-line coalesced global stores (box_out).  The other 190 KB
// or so go to the operand pipeline.
constexpr int kEpiBoxBytes = 4096;        // plain epilogues
constexpr int kEpiBoxBytesFused = 8192;   // fused epilogues (drain_fused's slots)
constexpr int kSmemLimit = 232448;        // 227 KB per CTA
constexpr int kMaxStages = 8;             // barrier slots reserved
// operand stages that fit beside the epilogue boxes, the barriers and the
// 1 KB alignment slack
constexpr int stages_for(int stage_bytes, int box_bytes) {
  return (kSmemLimit - 1024 - 512 - kEpiWarps * box_bytes) / stage_bytes < kMaxStages
             ? (kSmemLimit - 1024 - 512 - kEpiWarps * box_bytes) / stage_bytes
             : kMaxStages;
}

template <int BN>
struct Cfg {
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kBarrierBytes = 512;
  static int smem(int nst, int box) { return nst * kStageBytes + kEpiWarps * box + kBarrierBytes + 1024; }
};

// HAP_GEMM_TRACE builds (tools/gemm_trace.py): per-CTA %globaltimer stamps
// of the pipeline's milestones, to see where a launch's fixed cost goes.
constexpr int kTraceSlots = 32;
#ifdef HAP_GEMM_TRACE
__device__ unsigned long long* g_trace = nullptr;
__device__ int g_trace_ctas = 0;
__device__ __forceinline__ void trace(int ev) {
  if (g_trace && static_cast<int>(blockIdx.x) < g_trace_ctas) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_trace[blockIdx.x * kTraceSlots + ev] = t;
  }
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void trace_put(int ev, unsigned long long v) {
  if (g_trace && static_cast<int>(blockIdx.x) < g_trace_ctas) g_trace[blockIdx.x * kTraceSlots + ev] = v;
}
__device__ __forceinline__ void trace_add(int ev, unsigned long long v) {
  if (g_trace && static_cast<int>(blockIdx.x) < g_trace_ctas) g_trace[blockIdx.x * kTraceSlots + ev] += v;
}
// time spent in one wait, accumulated into `acc` (ns)
#define HAP_TIMED(acc, stmt) do { const unsigned long long t_ = gtimer(); stmt; (acc) += gtimer() - t_; } while (0)
#define HAP_TRACE(ev) trace(ev)
#define HAP_TRACE_ONCE(ev, flag) do { if (!(flag)) { trace(ev); (flag) = true; } } while (0)
// epilogue step timing of one warp (quarter 0, half 0, lane 0) into slot ev
#define HAP_ETIMED(on, ev, stmt) do { const unsigned long long t_ = gtimer(); stmt; if (on) trace_add(ev, gtimer() - t_); } while (0)
#else
#define HAP_ETIMED(on, ev, stmt) stmt
#define HAP_TIMED(acc, stmt) stmt
#define HAP_TRACE_ONCE(ev, flag) ((void)0)
#define HAP_TRACE(ev) ((void)0)
#endif

// ------------------------------------------------------------------ PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                            int32_t x, int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   bar)
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),
        "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor, 128B swizzle, sm_100 version field.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) |
         (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}

// Instruction descriptor: bf16 x bf16 -> fp32, M x N, operand major-ness.
__host__ __device__ constexpr uint32_t idesc(int m, int n, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

template <typename OutT>
__device__ __forceinline__ void store_row_chunk(OutT* dst, const uint32_t (&r)[32], int valid,
                                                bool vec, int accumulate) {
  if constexpr (std::is_same<OutT, float>::value) {
    if (vec && valid == 32) {
      float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 v = make_float4(__uint_as_float(r[4 * i]), __uint_as_float(r[4 * i + 1]),
                               __uint_as_float(r[4 * i + 2]), __uint_as_float(r[4 * i + 3]));
        if (accumulate) {
          float4 o = d4[i];
          v.x += o.x; v.y += o.y; v.z += o.z; v.w += o.w;
        }
        d4[i] = v;
      }
    } else {
      for (int i = 0; i < valid; ++i) {
        float v = __uint_as_float(r[i]);
        dst[i] = accumulate ? dst[i] + v : v;
      }
    }
  } else {
    if (vec && valid == 32) {
      uint4* d4 = reinterpret_cast<uint4*>(dst);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float f[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) f[j] = __uint_as_float(r[8 * i + j]);
        if (accumulate) {
          uint4 o = d4[i];
          const __nv_bfloat162* ob = reinterpret_cast<const __nv_bfloat162*>(&o);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float2 of = __bfloat1622float2(ob[j]);
            f[2 * j] += of.x;
            f[2 * j + 1] += of.y;
          }
        }
        uint4 v;
        __nv_bfloat162* vb = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
        for (int j = 0; j < 4; ++j) vb[j] = __floats2bfloat162_rn(f[2 * j], f[2 * j + 1]);
        d4[i] = v;
      }
    } else {
      for (int i = 0; i < valid; ++i) {
        float v = __uint_as_float(r[i]);
        if (accumulate) v += __bfloat162float(dst[i]);
        dst[i] = __float2bfloat16_rn(v);
      }
    }
  }
}

// stream-K helpers: a cut tile's fp32 partial, column-major [BN][128] per CTA
// (the TMEM lane = row is the fast index), so a warp's 32 lanes move one
// column as one coalesced 128-byte access.
__device__ __forceinline__ void add_partial(uint32_t (&r)[32], const float* p) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __ldcg(p + i * 128);
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) + v[i]);
}
template <int BN>
__device__ __forceinline__ void write_partial(uint32_t tmem_acc, int quarter, int half, int lane, float* part) {
  const uint32_t lane_base = tmem_acc + (static_cast<uint32_t>(quarter * 32) << 16) + half * (BN / 2);
  float* col0 = part + (half * (BN / 2)) * 128 + quarter * 32 + lane;
#pragma unroll 1
  for (int c = 0; c < BN / 64; ++c) {
    uint32_t r[32];
    tmem_ld32(lane_base + c * 32, r);
#pragma unroll
    for (int i = 0; i < 32; ++i) __stcg(col0 + (c * 32 + i) * 128, __uint_as_float(r[i]));
  }
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
// Before a CTA exits: its staged boxes have been read by the TMA engine (the
// global writes complete with the grid).
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// Every bulk store / reduce this thread committed has been performed in global memory.
__device__ __forceinline__ void bulk_wait_complete() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t src, int32_t x, int32_t y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y)
               : "memory");
}
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, uint32_t src, int32_t x, int32_t y) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y)
               : "memory");
}

// Epilogue modes: direct per-thread stores (any layout), TMA bulk store, TMA
// bulk reduce-add (fp32 accumulate: one writer per element), and split K
// (EPI_SPLIT_WS): each K split stores its fp32 partial tile into its own
// slice of a per-stream workspace, and split_reduce_kernel then sums the
// slices in split order and applies accumulate / the residual epilogue —
// deterministic (no floating-point atomics), with no dependency between the
// GEMM's CTAs (a split GEMM can share the GPU with spinning peer-memory
// kernels on other streams without deadlock).
enum { EPI_DIRECT = 0, EPI_TMA_STORE = 1, EPI_TMA_ADD = 2, EPI_SPLIT_WS = 3 };
// fused elementwise ops of the epilogue (hap_gemm_desc.epi)
enum { EPI_OP_NONE = HAP_EPI_NONE, EPI_OP_ADD = HAP_EPI_ADD, EPI_OP_ADD2 = HAP_EPI_ADD2,
       EPI_OP_SWISH = HAP_EPI_SWISH, EPI_OP_SWISH_BWD = HAP_EPI_SWISH_BWD };

// Byte offset of 16-byte chunk c of row r in a TMA-swizzled staging box.
template <int kRowBytes>
__device__ __forceinline__ uint32_t swz_offset(int r, int c) {
  if constexpr (kRowBytes == 128) return r * 128 + ((c ^ (r & 7)) << 4);
  else return r * 64 + ((c ^ ((r >> 1) & 3)) << 4);
}

__device__ __forceinline__ void red_add_v4(float* p, const uint32_t (&q)[4]) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(__uint_as_float(q[0])),
               "f"(__uint_as_float(q[1])), "f"(__uint_as_float(q[2])), "f"(__uint_as_float(q[3]))
               : "memory");
}

// Copy one staged 32-row box (rows of kRowBytes, swizzled 16-byte chunks) to
// global memory with full-line coalesced accesses: per pass, CPR consecutive
// lanes cover one row, the warp 32 / CPR rows.  kAdd (fp32 accumulate):
// vector reduce-add — one writer per element, so the result is the same
// whatever the order.  Rows >= M and columns >= N are not written.
template <typename OutT, int kRowBytes, bool kAdd>
__device__ __forceinline__ void box_out(uint32_t box, int lane, OutT* C, int64_t ldc, int row0, int col0, int M,
                                        int N, int vec_ok) {
  constexpr int CPR = kRowBytes / 16;
  constexpr int EPC = 16 / static_cast<int>(sizeof(OutT));
  constexpr int RPP = 32 / CPR;
#pragma unroll
  for (int it = 0; it < CPR; ++it) {
    const int r = it * RPP + lane / CPR, c = lane % CPR;
    uint32_t q[4];
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3])
                 : "r"(box + swz_offset<kRowBytes>(r, c)));
    const int row = row0 + r, col = col0 + c * EPC;
    if (row >= M || col >= N) continue;
    OutT* dst = C + static_cast<int64_t>(row) * ldc + col;
    if (vec_ok && col + EPC <= N) {
      if constexpr (kAdd) red_add_v4(reinterpret_cast<float*>(dst), q);
      else *reinterpret_cast<uint4*>(dst) = make_uint4(q[0], q[1], q[2], q[3]);
    } else {
      const OutT* v = reinterpret_cast<const OutT*>(q);
      const int valid = N - col < EPC ? N - col : EPC;
      for (int e = 0; e < valid; ++e) {
        if constexpr (kAdd) dst[e] = static_cast<float>(dst[e]) + static_cast<float>(v[e]);
        else dst[e] = v[e];
      }
    }
  }
}

// Drain one warp's 32 rows x BN/2 columns of a finished accumulator.
// TMA modes stage 32 x 128 B boxes (64 bf16 or 32 fp32 columns) in a
// 128B-swizzled double buffer — 16-byte chunk c of row r at c ^ (r & 7), the
// TMA SWIZZLE_128B pattern, which spreads a warp's 16 B stores over all banks —
// and hand each box to the TMA engine, so global writes are full lines issued
// asynchronously instead of 32 scattered row segments per store instruction.
template <int BN, typename OutT>
__device__ __forceinline__ void drain_accumulator(uint32_t tmem_acc, int quarter, int half, int lane, int row0,
                                                  int col0, int M, int N, OutT* C, int64_t ldc, int mode,
                                                  int vec_ok, int accumulate,
                                                  const CUtensorMap* tmC, uint8_t* buf, uint32_t& box_seq,
                                                  const float* prow = nullptr) {
  const uint32_t lane_base = tmem_acc + (static_cast<uint32_t>(quarter * 32) << 16);
  const int first = col0 + half * (BN / 2);
  if (mode == EPI_DIRECT) {
    const int row = row0 + lane;
    OutT* crow = C + static_cast<int64_t>(row) * ldc;
#pragma unroll 1
    for (int c = 0; c < BN / 64; ++c) {
      uint32_t r[32];
      tmem_ld32(lane_base + half * (BN / 2) + c * 32, r);
      const int col = first + c * 32;
      const int valid = N - col < 32 ? N - col : 32;
      if (row < M && valid > 0) store_row_chunk<OutT>(crow + col, r, valid, vec_ok, accumulate);
    }
    return;
  }
  // Box rows of 128 B when the warp's BN/2 columns split into them evenly,
  // else 64 B rows; 16-byte chunk c of row r is stored at the swizzled
  // position (swz_offset) so the row-per-lane writes and the row-major reads
  // of box_out both hit every bank.
  constexpr int kWide = 128 / static_cast<int>(sizeof(OutT));
  constexpr int W = ((BN / 2) % kWide == 0) ? kWide : kWide / 2;   // columns per box
  constexpr int kRowBytes = W * static_cast<int>(sizeof(OutT));
  constexpr int kBoxes = (BN / 2) / W;
  const uint32_t box = smem_u32(buf);
  const bool tr = quarter == 0 && half == 0 && lane == 0;
  (void)tr;
  (void)box_seq;
  (void)tmC;
#pragma unroll 1
  for (int b = 0; b < kBoxes; ++b) {
#ifdef HAP_GEMM_TRACE
    if (tr) trace_add(20, 1);
    const unsigned long long t_st = gtimer();
#endif
#pragma unroll
    for (int k = 0; k < W / 32; ++k) {
      uint32_t r[32];
      HAP_ETIMED(tr, 17, tmem_ld32(lane_base + half * (BN / 2) + b * W + k * 32, r));
      if (prow) add_partial(r, prow + (b * W + k * 32) * 128);
      if constexpr (std::is_same<OutT, float>::value) {
        static_assert(W % 32 == 0 || W == 16, "fp32 box width");
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t at = box + swz_offset<kRowBytes>(lane, j);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(at), "r"(r[4 * j]), "r"(r[4 * j + 1]),
                       "r"(r[4 * j + 2]), "r"(r[4 * j + 3]));
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t p[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            __nv_bfloat162 h = __floats2bfloat162_rn(__uint_as_float(r[8 * j + 2 * e]),
                                                     __uint_as_float(r[8 * j + 2 * e + 1]));
            p[e] = *reinterpret_cast<uint32_t*>(&h);
          }
          const uint32_t at = box + swz_offset<kRowBytes>(lane, k * 4 + j);
          asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(at), "r"(p[0]), "r"(p[1]), "r"(p[2]),
                       "r"(p[3]));
        }
      }
    }
    __syncwarp();
#ifdef HAP_GEMM_TRACE
    if (tr) trace_add(18, gtimer() - t_st);
    const unsigned long long t_o = gtimer();
#endif
    if (mode == EPI_TMA_ADD) {
      if constexpr (std::is_same<OutT, float>::value)
        box_out<float, kRowBytes, true>(box, lane, C, ldc, row0, first + b * W, M, N, vec_ok);
    } else {
      box_out<OutT, kRowBytes, false>(box, lane, C, ldc, row0, first + b * W, M, N, vec_ok);
    }
    __syncwarp();   // every lane has read the box before the next one is written
#ifdef HAP_GEMM_TRACE
    if (tr) trace_add(19, gtimer() - t_o);
#endif
  }
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ------------------------------------------------------------------ batched problems
// One persistent launch serves up to kMaxProblems GEMMs of the same operand
// orientation: either independent problems whose tiles share the launch
// (grouped: e.g. the Q/K/V projections of one input), or problems that all
// add into one output (sum_k: C = sum_i A_i . B_i, the K blocks of every
// problem accumulate into the same TMEM tile — e.g. dx = dq.Wq^T + dk.Wk^T +
// dv.Wv^T).  Small GEMMs pay the launch, prologue and partial last wave once.
constexpr int kMaxProblems = 4;

struct alignas(64) TcProblem {
  CUtensorMap a, b, c;     // c: output map (TMA epilogues)
  void* C;
  int64_t ldc;
  float* ws;               // EPI_SPLIT_WS: fp32 partials [splits][ws_rows][ws_ld]
  int64_t ws_ld;
  int ws_rows;             // rows per split slice (M rounded up to whole tiles)
  int M, N, K;
  int m_tiles, n_tiles, k_blocks;
  int splits, kb_per_split;
  int unit_begin;
  int epi_mode, accumulate, vec_ok;
  // fused epilogue (hap_gemm_desc.epi): two extra bf16 tensor maps with C's
  // box geometry, loaded into / stored from the staging boxes by TMA:
  //   ADD: e1 = R (in)   ADD2: e1 = R (in), e2 = Y (out)
  //   SWISH: e1 = Y, e2 = Z (out)   SWISH_BWD: e1 = R = x, e2 = R2 = f(x) (in)
  int epi, epi_tag;
  CUtensorMap e1, e2;
};

struct alignas(64) TcBatch {
  TcProblem p[kMaxProblems];
  // shared-memory layout of this launch: nst operand stages, then one
  // epilogue box of box_bytes per epilogue warp (4 KB; 8 KB when a fused
  // epilogue stages its TMA-loaded inputs and three-output chunks), then the
  // barriers — a plain launch turns the spare 32 KB into pipeline depth
  int nst, box_bytes;
  int count;
  int sum_k;
  int sum_kb;              // sum_k: K blocks of all problems (the concatenated K range)
  int total_units;
  // stream-K (SM-pair kernel, one problem): pair p walks K-block iterations
  // [p*I/P, (p+1)*I/P) of the I = tiles x k_blocks iteration space, so every
  // pair gets the same MMA work whatever the tile count; a tile cut by a range
  // boundary is finished by the pair holding its first K blocks, after adding
  // the fp32 partial of its last K blocks that the next pair wrote to slot
  // (boundary index) of the workspace.
  int sk;                  // 0: data-parallel units
  int sk_kb;               // K blocks per tile
  int sk_pairs;            // P
  long long sk_iters;      // I
  float* sk_ws;            // [P + 1][2 CTAs][128][BN] fp32 partial tiles
  unsigned* sk_flags;      // [P + 1][2 CTAs][8 epilogue warps]: partial written
  // cluster split K (single-CTA kernel): csplit > 1 CTAs of one thread-block
  // cluster share an output tile, CTA rank s walking the s-th slice of its K
  // blocks; their fp32 partials meet in distributed shared memory and every
  // CTA finishes 128 / csplit rows of the tile, adding the partials in rank
  // order (cluster_split_finish)
  int csplit;
  // the residual epilogue the finish applies per problem (NONE / ADD / ADD2)
  int fin_epi[kMaxProblems];
  const void* fin_R[kMaxProblems];
  void* fin_Y[kMaxProblems];
  int64_t fin_ldr[kMaxProblems], fin_ldy[kMaxProblems];
};

// Touch every 64-byte line of the launch parameters from one idle warp while
// the prologue runs: the unit decode of the producer, MMA and epilogue
// cursors reads TcBatch fields with dynamic indices (constant-cache loads),
// and their first, serialised misses otherwise sit between the prologue and
// the first TMA load (~0.6-1 us per launch, tools/gemm_trace.py).
__device__ __forceinline__ void warm_params(const TcBatch& bt, int lane) {
  const int* w = reinterpret_cast<const int*>(&bt);
  constexpr int kLines = (static_cast<int>(sizeof(TcBatch)) + 63) / 64;
  int acc = 0;
#pragma unroll
  for (int i = lane; i < kLines; i += 32) acc += w[i * 16];
  asm volatile("" ::"r"(acc));
}

__device__ __forceinline__ float bf16_round(float v) { return __bfloat162float(__float2bfloat16_rn(v)); }

// 8 consecutive fp32 accumulator columns of this warp's 32 TMEM lanes.
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(r[e]);
}

__device__ __forceinline__ void lds_bf16x8(uint32_t at, float (&v)[8]) {
  uint32_t q[4];
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]) : "r"(at));
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 f = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&q[e]));
    v[2 * e] = f.x;
    v[2 * e + 1] = f.y;
  }
}

__device__ __forceinline__ void sts_bf16x8(uint32_t at, const float (&v)[8]) {
  uint32_t p[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * e], v[2 * e + 1]);
    p[e] = *reinterpret_cast<uint32_t*>(&h);
  }
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(at), "r"(p[0]), "r"(p[1]), "r"(p[2]), "r"(p[3]));
}

__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

// Fused epilogues (hap_gemm_desc.epi, bf16 outputs).  The warp drains its
// 32 rows x BN/2 columns in chunks of 32 columns (one tcgen05.ld each); every
// tensor a chunk touches — outputs (C, Y, Z) and inputs (R, x, f(x)) — is a
// 32 x 32 bf16 box (64-byte rows, SWIZZLE_64B) in the warp's 8 KB staging area
// (4 slots of 2 KB).  Inputs are TMA-loaded into the slot their output will
// occupy and overwritten in place; outputs leave by TMA store, one bulk group
// per chunk.  Ops with <= 2 slots per chunk double-buffer: the next chunk's
// inputs are loaded into the other slot pair while this chunk computes.
// Rounding follows the unfused kernels: C is rounded to bf16 first and the
// elementwise results are computed from the rounded value (elementwise.cu
// swish_fwd / binary / swish_bwd).
constexpr int kFusedW = 32;                  // columns per fused box
constexpr int kFusedBox = 32 * kFusedW * 2;  // bytes per fused box

// bf16 rounding of two fp32 values at once: one F2FP pack (ALU pipe) and two
// shifts, the same round-to-nearest-even as __float2bfloat16_rn per value
// (F2F, a quarter-rate XU-pipe op that MUFU shares — with two of them per
// element and the sigmoid's two MUFU ops, the swish epilogue was XU-bound).
// Returns the packed pair (low = a) and replaces a, b by their rounded values.
__device__ __forceinline__ uint32_t round2_bf16(float& a, float& b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  const uint32_t u = *reinterpret_cast<const uint32_t*>(&h);
  a = __uint_as_float(u << 16);
  b = __uint_as_float(u & 0xffff0000u);
  return u;
}

__device__ __forceinline__ void sts_u32x4(uint32_t at, const uint32_t (&p)[4]) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(at), "r"(p[0]), "r"(p[1]), "r"(p[2]), "r"(p[3]));
}

// The elementwise op of one 32-column chunk: r = accumulator columns of the
// lane's row; s0..s2 = the chunk's staging slots (inputs in place, outputs).
// Values are rounded to bf16 exactly where the unfused kernels store them,
// two at a time (round2_bf16).
template <int EPI, int TAG>
__device__ __forceinline__ void fused_chunk(const uint32_t (&r)[32], int lane, uint32_t s0, uint32_t s1,
                                            uint32_t s2) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {   // 8 columns: 16-byte chunk j of the lane's 64-byte row
    const uint32_t off = swz_offset<64>(lane, j);
    float c[8], x[8], y[8];
    uint32_t p0[4], p1[4], p2[4];
#pragma unroll
    for (int e = 0; e < 8; ++e) c[e] = __uint_as_float(r[8 * j + e]);
    if constexpr (EPI == EPI_OP_ADD) {   // C = bf16(acc + R)
      lds_bf16x8(s0 + off, x);
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        float a = c[e] + x[e], b = c[e + 1] + x[e + 1];
        p0[e / 2] = round2_bf16(a, b);
      }
    } else if constexpr (EPI == EPI_OP_ADD2) {   // C = bf16(acc); Y = bf16(C + R)
      lds_bf16x8(s1 + off, x);
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        float a = c[e], b = c[e + 1];
        p0[e / 2] = round2_bf16(a, b);
        float u = a + x[e], v = b + x[e + 1];
        p1[e / 2] = round2_bf16(u, v);
      }
    } else if constexpr (EPI == EPI_OP_SWISH) {   // C = bf16(acc); Y = bf16(f(C)); Z = bf16(C * Y)
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        float a = c[e], b = c[e + 1];
        p0[e / 2] = round2_bf16(a, b);
        float ya = unary_fwd_t<TAG>(a), yb = unary_fwd_t<TAG>(b);
        p1[e / 2] = round2_bf16(ya, yb);
        float za = a * ya, zb = b * yb;
        p2[e / 2] = round2_bf16(za, zb);
      }
    } else {   // EPI_OP_SWISH_BWD: C = dz*y + (dz*x)*f'(x, y), dz = rounded accumulator
      lds_bf16x8(s0 + off, x);
      lds_bf16x8(s1 + off, y);
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        float ga = c[e], gb = c[e + 1];
        round2_bf16(ga, gb);
        float da = ga * x[e], db = gb * x[e + 1];
        round2_bf16(da, db);
        float ta = da * unary_deriv(TAG, x[e], y[e]), tb = db * unary_deriv(TAG, x[e + 1], y[e + 1]);
        round2_bf16(ta, tb);
        float oa = ga * y[e] + ta, ob = gb * y[e + 1] + tb;
        p0[e / 2] = round2_bf16(oa, ob);
      }
    }
    sts_u32x4(s0 + off, p0);
    if constexpr (EPI == EPI_OP_ADD2 || EPI == EPI_OP_SWISH) sts_u32x4(s1 + off, p1);
    if constexpr (EPI == EPI_OP_SWISH) sts_u32x4(s2 + off, p2);
  }
}

template <int BN>
__device__ __forceinline__ void drain_fused(const TcProblem& pr, uint32_t tmem_acc, int quarter, int half, int lane,
                                            int row0, int col0, uint8_t* buf, uint32_t ld_bar0, uint32_t& ld_phase,
                                            const float* prow) {
  constexpr int kChunks = (BN / 2) / kFusedW;
  const uint32_t lane_base = tmem_acc + (static_cast<uint32_t>(quarter * 32) << 16) + half * (BN / 2);
  const int first = col0 + half * (BN / 2);
  const int epi = pr.epi;
  const int n_in = epi == EPI_OP_SWISH_BWD ? 2 : ((epi == EPI_OP_ADD || epi == EPI_OP_ADD2) ? 1 : 0);
  const bool dbl = epi != EPI_OP_SWISH;   // <= 2 slots per chunk: two slot pairs alternate
  const uint32_t buf0 = smem_u32(buf);
  // slot of input i / output o in slot set `set`
  // dbl: slot pair `set`; otherwise (three outputs per chunk) `set` is the
  // chunk index and its boxes take the next three slots of a 4-slot ring
  auto slot = [&](int set, int k) -> uint32_t {
    return buf0 + (dbl ? set * 2 + k : ((3 * set + k) & 3)) * kFusedBox;
  };
  auto in_slot = [&](int set, int i) -> uint32_t { return slot(set, epi == EPI_OP_ADD2 ? 1 : i); };
  auto issue_loads = [&](int chunk) {   // lane 0
    const int set = dbl ? (chunk & 1) : 0;
    const uint32_t bar = ld_bar0 + 8 * set;
    mbar_expect_tx(bar, n_in * kFusedBox);
    const int x0 = first + chunk * kFusedW;
    tma_load_2d(in_slot(set, 0), &pr.e1, bar, x0, row0);
    if (n_in == 2) tma_load_2d(in_slot(set, 1), &pr.e2, bar, x0, row0);
  };
  fence_async_smem();   // a preceding plain unit's generic accesses to this box come first
  __syncwarp();
  if (lane == 0) {
    bulk_wait_read0();   // the previous unit's stores have read the staging slots
    if (n_in) issue_loads(0);
  }
  __syncwarp();
  const bool tr = quarter == 0 && half == 0 && lane == 0;
  (void)tr;
#pragma unroll 1
  for (int ch = 0; ch < kChunks; ++ch) {
    const int set = dbl ? (ch & 1) : ch;
#ifdef HAP_GEMM_TRACE
    if (tr) trace_add(26, 1);
    const unsigned long long t_w = gtimer();
#endif
    if (lane == 0) {
      if (dbl) {
        // the other pair was last stored from by chunk ch-1: once read out,
        // prefetch chunk ch+1's inputs into it
        if (ch + 1 < kChunks) {
          bulk_wait_read0();
          if (n_in) issue_loads(ch + 1);
        }
      } else {
        bulk_wait_read1();   // ring: only the previous chunk's last box may still be read
      }
    }
#ifdef HAP_GEMM_TRACE
    if (tr) trace_add(22, gtimer() - t_w);
#endif
    uint32_t r[32];
    HAP_ETIMED(tr, 23, tmem_ld32(lane_base + ch * kFusedW, r));
    if (prow) add_partial(r, prow + ch * kFusedW * 128);
    if (n_in) {
      HAP_ETIMED(tr, 21, mbar_wait(ld_bar0 + 8 * set, (ld_phase >> set) & 1));
      ld_phase ^= 1u << set;
    }
    __syncwarp();
#ifdef HAP_GEMM_TRACE
    const unsigned long long t_c = gtimer();
#endif
    const uint32_t s0 = slot(set, 0), s1 = slot(set, 1), s2 = slot(set, 2);
    // one dispatch per chunk: the 32 columns run a loop specialised on (op, f)
#define HAP_FUSED_CASE(EPI, TAG) fused_chunk<EPI, TAG>(r, lane, s0, s1, s2)
    if (epi == EPI_OP_ADD) HAP_FUSED_CASE(EPI_OP_ADD, 0);
    else if (epi == EPI_OP_ADD2) HAP_FUSED_CASE(EPI_OP_ADD2, 0);
    else if (epi == EPI_OP_SWISH) {
      switch (pr.epi_tag) {
        case HAP_SIGMOID: HAP_FUSED_CASE(EPI_OP_SWISH, HAP_SIGMOID); break;
        case HAP_EXP: HAP_FUSED_CASE(EPI_OP_SWISH, HAP_EXP); break;
        case HAP_NEG: HAP_FUSED_CASE(EPI_OP_SWISH, HAP_NEG); break;
        case HAP_RELU: HAP_FUSED_CASE(EPI_OP_SWISH, HAP_RELU); break;
        default: HAP_FUSED_CASE(EPI_OP_SWISH, HAP_TANH); break;
      }
    } else {
      switch (pr.epi_tag) {
        case HAP_SIGMOID: HAP_FUSED_CASE(EPI_OP_SWISH_BWD, HAP_SIGMOID); break;
        case HAP_EXP: HAP_FUSED_CASE(EPI_OP_SWISH_BWD, HAP_EXP); break;
        case HAP_NEG: HAP_FUSED_CASE(EPI_OP_SWISH_BWD, HAP_NEG); break;
        case HAP_RELU: HAP_FUSED_CASE(EPI_OP_SWISH_BWD, HAP_RELU); break;
        default: HAP_FUSED_CASE(EPI_OP_SWISH_BWD, HAP_TANH); break;
      }
    }
#undef HAP_FUSED_CASE
    fence_async_smem();
    __syncwarp();
#ifdef HAP_GEMM_TRACE
    if (tr) trace_add(24, gtimer() - t_c);
    const unsigned long long t_i = gtimer();
#endif
    if (lane == 0) {
      const int x0 = first + ch * kFusedW;
      tma_store_2d(&pr.c, slot(set, 0), x0, row0);
      if (epi == EPI_OP_ADD2) tma_store_2d(&pr.e2, slot(set, 1), x0, row0);
      if (epi == EPI_OP_SWISH) {   // one bulk group per box (ring slots free up one by one)
        bulk_commit();
        tma_store_2d(&pr.e1, slot(set, 1), x0, row0);
        bulk_commit();
        tma_store_2d(&pr.e2, slot(set, 2), x0, row0);
      }
      bulk_commit();
    }
#ifdef HAP_GEMM_TRACE
    if (tr) trace_add(25, gtimer() - t_i);
#endif
  }
  // a following unit may be unfused: its staging boxes overlap these slots
  if (lane == 0) bulk_wait_read0();
  __syncwarp();
}

// Epilogue of one unit for one warp: drain the accumulator into C, or (split
// K) into split `split`'s slice of the workspace.
template <int BN, typename OutT>
__device__ __forceinline__ void epilogue_unit(const TcProblem& pr, uint32_t tmem_acc, int quarter, int half,
                                              int lane, int row0, int col0, int split, uint8_t* buf,
                                              uint32_t& box_seq, uint32_t ld_bar, uint32_t& ld_phase,
                                              const float* part) {
  // part: stream-K partial of this CTA's 128 x BN share (column-major), added to
  // the accumulator before anything is rounded
  const float* prow = part ? part + (half * (BN / 2)) * 128 + quarter * 32 + lane : nullptr;
  if constexpr (std::is_same<OutT, __nv_bfloat16>::value) {
    if (pr.epi != EPI_OP_NONE) {
      drain_fused<BN>(pr, tmem_acc, quarter, half, lane, row0, col0, buf, ld_bar, ld_phase, prow);
      return;
    }
  }
  if (pr.epi_mode == EPI_SPLIT_WS) {   // split s's slice: rows [s * ws_rows, s * ws_rows + M)
    drain_accumulator<BN, float>(tmem_acc, quarter, half, lane, split * pr.ws_rows + row0, col0,
                                 split * pr.ws_rows + pr.M, pr.N, pr.ws, pr.ws_ld, EPI_TMA_STORE, 1, 0, &pr.c, buf,
                                 box_seq);
    return;
  }
  drain_accumulator<BN, OutT>(tmem_acc, quarter, half, lane, row0, col0, pr.M, pr.N, static_cast<OutT*>(pr.C),
                              pr.ldc, pr.epi_mode, pr.vec_ok, pr.accumulate, &pr.c, buf, box_seq, prow);
}

struct Unit {
  int prob, split, tile, m0, n0, kb0, kb1;
  int sk_kind;   // 0: whole tile; 1: a tile's last K blocks (write partial); 2: its first (finish it)
  int sk_slot;   // workspace slot of a cut tile
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_cta(uint32_t addr, uint32_t cta) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(addr), "r"(cta));
  return out;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// ---- cluster split K (single-CTA kernel, TcBatch.csplit = S > 1)
// Each CTA of the tile's cluster drains its 128 x BN fp32 accumulator into
// its own (now idle) pipeline shared memory, row-major with the 16-byte
// chunks of row r XOR-swizzled by (r & 7) (a warp's 32 rows hit all banks).
// After a cluster barrier CTA s reduces rows [s * 128 / S, (s + 1) * 128 / S):
// every float4 chunk is read from all S CTAs' shared memory through DSMEM
// (mapa) and summed in rank order 0..S-1 — the same bits whatever the
// timing — then + C when accumulating, the residual epilogue with the
// unfused roundings (ADD: C = bf16(sum + R); ADD2: C = bf16(sum),
// Y = bf16(bf16(sum) + R)), and stored.  A second cluster barrier keeps every
// CTA's shared memory alive until all have read it.  The hardware schedules
// a cluster's CTAs together, so these waits need no co-residency beyond the
// cluster (unlike a grid-wide split finish).
__device__ __forceinline__ uint32_t csplit_offset(int row, int chunk, int bn) {
  return static_cast<uint32_t>(row * bn * 4 + ((chunk ^ (row & 7)) << 4));
}

// fp32 outputs (weight gradients): the splits of a tile add into C one after
// another in rank order — split s waits on its warp's turn barrier until
// split s-1 has finished, then drains its accumulator into C by TMA
// reduce-add (split 0 without accumulate: TMA store), waits until those
// writes are performed, and passes the turn to split s+1 (a release arrive
// on the next CTA's barrier, through the cluster).  C = ((C + p0) + p1) + ...
// on every run, at the price of the serialised adds (one tile slab each).
__device__ __forceinline__ void chain_wait(uint32_t bar) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "CHAINW_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 done, [%0], 0;\n\t"
      "@!done bra CHAINW_%=;\n}" ::"r"(bar)
      : "memory");
}
__device__ __forceinline__ void chain_pass(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}

template <int BN>
__device__ __forceinline__ void csplit_chain(const TcProblem& pr, const Unit& x, uint32_t tmem_acc, int quarter,
                                             int half, int lane, int row0, uint8_t* buf, uint32_t& box_seq,
                                             uint32_t turn, int next_rank) {
  if (x.split > 0) {
    if (lane == 0) chain_wait(turn);
    __syncwarp();
    asm volatile("fence.proxy.async.global;" ::: "memory");   // the acquire orders this warp's TMA reduce
  }
  const bool tma = pr.epi_mode == EPI_TMA_ADD;
  const int mode = tma ? ((x.split == 0 && !pr.accumulate) ? EPI_TMA_STORE : EPI_TMA_ADD) : EPI_DIRECT;
  drain_accumulator<BN, float>(tmem_acc, quarter, half, lane, row0, x.n0, pr.M, pr.N, static_cast<float*>(pr.C),
                               pr.ldc, mode, pr.vec_ok, (x.split > 0 || pr.accumulate) ? 1 : 0, &pr.c, buf,
                               box_seq);
  __threadfence();   // this lane's adds into C are performed before the turn passes
  __syncwarp();
  if (next_rank >= 0 && lane == 0) chain_pass(map_to_cta(turn, static_cast<uint32_t>(next_rank)));
}

template <int BN>
__device__ __forceinline__ void csplit_drain(uint32_t tmem_acc, int quarter, int half, int lane, uint8_t* part,
                                             bool empty) {
  const int row = quarter * 32 + lane;
  const uint32_t lane_base = tmem_acc + (static_cast<uint32_t>(quarter * 32) << 16) + half * (BN / 2);
  const uint32_t base = smem_u32(part);
#pragma unroll 1
  for (int c = 0; c < BN / 64; ++c) {
    uint32_t r[32];
    if (empty) {
#pragma unroll
      for (int i = 0; i < 32; ++i) r[i] = 0u;   // an empty K slice contributes zeros
    } else {
      tmem_ld32(lane_base + c * 32, r);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int chunk = (half * (BN / 2) + c * 32) / 4 + j;
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + csplit_offset(row, chunk, BN)),
                   "r"(r[4 * j]), "r"(r[4 * j + 1]), "r"(r[4 * j + 2]), "r"(r[4 * j + 3]));
    }
  }
}

__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t cluster_addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(cluster_addr)
               : "memory");
  return v;
}

// `rank` = this CTA's index among the S that hold the same rows, whose
// cluster ranks are q * stride + offset (single-CTA tiles: stride 1; SM-pair
// tiles: stride 2, offset = rank within the pair).  16 DSMEM loads (16 / S
// chunks x S partials) plus their C / R loads are in flight per iteration.
template <int BN, typename OutT, int S>
__device__ __forceinline__ void csplit_finish_t(const TcBatch& bt, const TcProblem& pr, int prob, int m0, int n0,
                                                uint8_t* part, int rank, int tid, int stride, int offset) {
  constexpr int kChunks = BN / 4;   // float4 chunks per row
  constexpr int CPI = 16 / S;       // chunks per iteration per thread
  constexpr int kThreadsE = kEpiWarps * 32;
  const int rows = 128 / S;
  const int r0 = rank * rows;
  const int total = rows * kChunks;
  const uint32_t base = smem_u32(part);
  uint32_t peer[S];
#pragma unroll
  for (int q = 0; q < S; ++q) peer[q] = map_to_cta(base, static_cast<uint32_t>(q * stride + offset));
  const int epi = bt.fin_epi[prob];
  const bool acc_c = pr.accumulate != 0;
  for (int k0 = tid; k0 < total; k0 += CPI * kThreadsE) {
    float4 v[CPI][S];
#pragma unroll
    for (int c = 0; c < CPI; ++c) {
      const int k = k0 + c * kThreadsE;
      if (k < total) {
        const uint32_t off = csplit_offset(r0 + k / kChunks, k % kChunks, BN);
#pragma unroll
        for (int q = 0; q < S; ++q) v[c][q] = ld_dsmem_f4(peer[q] + off);
      }
    }
    float old[CPI][4], res[CPI][4];
#pragma unroll
    for (int c = 0; c < CPI; ++c) {
      const int k = k0 + c * kThreadsE;
#pragma unroll
      for (int j = 0; j < 4; ++j) old[c][j] = res[c][j] = 0.f;
      if (k >= total) continue;
      const int grow = m0 + r0 + k / kChunks, col = n0 + (k % kChunks) * 4;
      if (grow >= pr.M || col >= pr.N) continue;
      const int valid = pr.N - col < 4 ? pr.N - col : 4;
      const OutT* dst = static_cast<const OutT*>(pr.C) + static_cast<int64_t>(grow) * pr.ldc + col;
      if (acc_c) {
        if constexpr (std::is_same<OutT, float>::value) {
          if (valid == 4 && pr.vec_ok) {
            const float4 o = *reinterpret_cast<const float4*>(dst);
            old[c][0] = o.x; old[c][1] = o.y; old[c][2] = o.z; old[c][3] = o.w;
          } else {
            for (int j = 0; j < valid; ++j) old[c][j] = dst[j];
          }
        } else {
          for (int j = 0; j < valid; ++j) old[c][j] = __bfloat162float(dst[j]);
        }
      }
      if (epi != EPI_OP_NONE) {
        const __nv_bfloat16* R = static_cast<const __nv_bfloat16*>(bt.fin_R[prob]) +
                                 static_cast<int64_t>(grow) * bt.fin_ldr[prob] + col;
        for (int j = 0; j < valid; ++j) res[c][j] = __bfloat162float(R[j]);
      }
    }
#pragma unroll
    for (int c = 0; c < CPI; ++c) {
      const int k = k0 + c * kThreadsE;
      if (k >= total) continue;
      const int grow = m0 + r0 + k / kChunks, col = n0 + (k % kChunks) * 4;
      if (grow >= pr.M || col >= pr.N) continue;
      float4 a = v[c][0];
#pragma unroll
      for (int q = 1; q < S; ++q) {   // rank order: the same sum whatever the timing
        a.x += v[c][q].x; a.y += v[c][q].y; a.z += v[c][q].z; a.w += v[c][q].w;
      }
      float f[4] = {a.x + old[c][0], a.y + old[c][1], a.z + old[c][2], a.w + old[c][3]};
      const int valid = pr.N - col < 4 ? pr.N - col : 4;
      OutT* dst = static_cast<OutT*>(pr.C) + static_cast<int64_t>(grow) * pr.ldc + col;
      if constexpr (std::is_same<OutT, float>::value) {
        if (valid == 4 && pr.vec_ok) *reinterpret_cast<float4*>(dst) = make_float4(f[0], f[1], f[2], f[3]);
        else for (int j = 0; j < valid; ++j) dst[j] = f[j];
      } else {
        if (epi == EPI_OP_ADD)
          for (int j = 0; j < 4; ++j) f[j] += res[c][j];
        for (int j = 0; j < valid; ++j) dst[j] = __float2bfloat16_rn(f[j]);
        if (epi == EPI_OP_ADD2) {
          __nv_bfloat16* Y = static_cast<__nv_bfloat16*>(bt.fin_Y[prob]) +
                             static_cast<int64_t>(grow) * bt.fin_ldy[prob] + col;
          for (int j = 0; j < valid; ++j) Y[j] = __float2bfloat16_rn(bf16_round(f[j]) + res[c][j]);
        }
      }
    }
  }
}

template <int BN, typename OutT>
__device__ __forceinline__ void csplit_finish(const TcBatch& bt, const TcProblem& pr, int prob, int m0, int n0,
                                              uint8_t* part, int rank, int S, int tid, int stride = 1,
                                              int offset = 0) {
  switch (S) {
    case 2: csplit_finish_t<BN, OutT, 2>(bt, pr, prob, m0, n0, part, rank, tid, stride, offset); break;
    case 4: csplit_finish_t<BN, OutT, 4>(bt, pr, prob, m0, n0, part, rank, tid, stride, offset); break;
    default: csplit_finish_t<BN, OutT, 8>(bt, pr, prob, m0, n0, part, rank, tid, stride, offset); break;
  }
}

// Work unit u -> (problem, output tile, K-block range).  Grouped: units are
// laid out problem after problem; within a problem unit = split * tiles + tile.
template <int ROWS, int BN>
__device__ __forceinline__ Unit decode_unit(const TcBatch& bt, int u) {
  const int S = bt.csplit > 1 ? bt.csplit : 1;
  const int cs = u % S;   // cluster split: CTA rank within the tile's cluster
  u /= S;
  int p = 0;
  if (!bt.sum_k)
    while (p + 1 < bt.count && u >= bt.p[p + 1].unit_begin) ++p;
  const TcProblem& pr = bt.p[p];
  const int local = u - pr.unit_begin;
  const int tiles = pr.m_tiles * pr.n_tiles;
  const int t = local % tiles;
  Unit x;
  x.prob = p;
  x.split = local / tiles;
  x.tile = t;
  x.m0 = (t % pr.m_tiles) * ROWS;
  x.n0 = (t / pr.m_tiles) * BN;
  x.kb0 = (local / tiles) * pr.kb_per_split;
  x.kb1 = min(bt.sum_k ? bt.sum_kb : pr.k_blocks, x.kb0 + pr.kb_per_split);
  if (S > 1) {
    const int kb = bt.sum_k ? bt.sum_kb : pr.k_blocks;
    const int per = (kb + S - 1) / S;
    x.split = cs;
    x.kb0 = min(kb, cs * per);
    x.kb1 = min(kb, x.kb0 + per);
  }
  return x;
}

// The units one SM pair walks, in order: every num_pairs-th data-parallel
// unit, or (stream-K) the pieces of its iteration range.  Producer, MMA issuer
// and epilogue each run their own cursor and see the same sequence.
template <int BN>
struct PairCursor {
  long long it = 0, end = 0;
  int u = 0, step = 1, pair = 0;
  __device__ PairCursor(const TcBatch& bt, int pair_, int num_pairs) : pair(pair_) {
    if (bt.sk) {
      it = static_cast<long long>(pair) * bt.sk_iters / bt.sk_pairs;
      end = static_cast<long long>(pair + 1) * bt.sk_iters / bt.sk_pairs;
    } else {
      u = pair;
      step = num_pairs;
    }
  }
  __device__ bool next(const TcBatch& bt, Unit& x) {
    if (!bt.sk) {
      if (u >= bt.total_units) return false;
      x = decode_unit<256, BN>(bt, u);
      x.sk_kind = 0;
      x.sk_slot = 0;
      u += step;
      return true;
    }
    if (it >= end) return false;
    const TcProblem& pr = bt.p[0];
    const int kb = bt.sk_kb;
    const int tile = static_cast<int>(it / kb);
    const int kb0 = static_cast<int>(it - static_cast<long long>(tile) * kb);
    const int kb1 = static_cast<int>(min(static_cast<long long>(kb), kb0 + (end - it)));
    x.prob = 0;
    x.split = 0;
    x.tile = tile;
    x.m0 = (tile % pr.m_tiles) * 256;
    x.n0 = (tile / pr.m_tiles) * BN;
    x.kb0 = kb0;
    x.kb1 = kb1;
    x.sk_kind = (kb0 == 0 && kb1 == kb) ? 0 : (kb1 == kb ? 1 : 2);
    x.sk_slot = x.sk_kind == 1 ? pair : pair + 1;
    it += kb1 - kb0;
    return true;
  }
};

// f(problem, k_block) for every K block a unit accumulates, in order (a sum
// walks its slice [kb0, kb1) of the problems' concatenated K blocks).
template <typename F>
__device__ __forceinline__ void for_each_kblock(const TcBatch& bt, const Unit& x, F&& f) {
  if (bt.sum_k) {
    int base = 0;
    for (int q = 0; q < bt.count; ++q) {
      const int nk = bt.p[q].k_blocks;
      const int lo = max(x.kb0 - base, 0), hi = min(x.kb1 - base, nk);
      for (int kb = lo; kb < hi; ++kb) f(q, kb);
      base += nk;
    }
  } else {
    for (int kb = x.kb0; kb < x.kb1; ++kb) f(x.prob, kb);
  }
}

template <int BN, bool kAMN, bool kBMN, typename OutT>
__global__ void __launch_bounds__(kThreads, 1) gemm_tc_kernel(const __grid_constant__ TcBatch bt) {
  using G = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int nst = bt.nst;
  uint8_t* staging = smem + nst * G::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + kEpiWarps * bt.box_bytes);
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = smem_u32(bars + nst);
  const uint32_t tfull0 = smem_u32(bars + 2 * nst);
  const uint32_t tempty0 = smem_u32(bars + 2 * nst + 2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * nst + 4);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_units = bt.total_units;

  if (warp == 0 && lane == 0) {
    for (int q = 0; q < bt.count; ++q) {
      tma_prefetch(&bt.p[q].a);
      tma_prefetch(&bt.p[q].b);
    }
  }
  if (warp == 3) warm_params(bt, lane);
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull0 + 8 * a, 1);
      mbar_init(tempty0 + 8 * a, kEpiWarps * 32);
    }
    for (int w = 0; w < 2 * kEpiWarps; ++w) mbar_init(smem_u32(bars + 2 * nst + 6 + w), 1);
    for (int w = 0; w < kEpiWarps; ++w) mbar_init(smem_u32(bars + 2 * nst + 22 + w), 1);   // split-K turns
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(G::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  hap::pdl_wait();   // everything above touched no global memory

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        const Unit x = decode_unit<BM, BN>(bt, u);
        for_each_kblock(bt, x, [&](int q, int kb) {
          mbar_wait(empty0 + 8 * stage, phase ^ 1);
          const uint32_t fb = full0 + 8 * stage;
          mbar_expect_tx(fb, G::kStageBytes);
          const uint32_t sa = smem_u32(smem + stage * G::kStageBytes);
          const uint32_t sb = sa + G::kABytes;
          const int k0 = kb * BK;
          const CUtensorMap* ma = &bt.p[q].a;
          const CUtensorMap* mb = &bt.p[q].b;
          if (kAMN) {
            tma_load_2d(sa, ma, fb, x.m0, k0);
            tma_load_2d(sa + BK * 128, ma, fb, x.m0 + 64, k0);
          } else {
            tma_load_2d(sa, ma, fb, k0, x.m0);
          }
          if (kBMN) {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c) tma_load_2d(sb + c * BK * 128, mb, fb, x.n0 + 64 * c, k0);
          } else {
            tma_load_2d(sb, mb, fb, k0, x.n0);
          }
          if (++stage == nst) {
            stage = 0;
            phase ^= 1;
          }
        });
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t kIdesc = idesc(BM, BN, kAMN, kBMN);
      // K-major: rows of 128B, 8-row atoms 1024B apart (SBO), LBO unused (16B).
      // MN-major: K-rows of 128B, 8-row groups 1024B apart (SBO); successive
      // 64-element MN chunks BK*128 bytes apart (LBO).
      constexpr uint32_t kALbo = kAMN ? BK * 128 : 16;
      constexpr uint32_t kBLbo = kBMN ? BK * 128 : 16;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
        const Unit x = decode_unit<BM, BN>(bt, u);
        mbar_wait(tempty0 + 8 * acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        bool first = true;
        for_each_kblock(bt, x, [&](int, int) {
          mbar_wait(full0 + 8 * stage, phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * G::kStageBytes);
          const uint32_t sb = sa + G::kABytes;
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; ++kk) {
            const uint32_t aoff = kAMN ? kk * UMMA_K * 128 : kk * UMMA_K * 2;
            const uint32_t boff = kBMN ? kk * UMMA_K * 128 : kk * UMMA_K * 2;
            tc_mma(d_tmem, sdesc(sa + aoff, kALbo, 1024), sdesc(sb + boff, kBLbo, 1024), kIdesc,
                   (!first) || (kk != 0));
          }
          first = false;
          tc_commit(empty0 + 8 * stage);
          if (++stage == nst) {
            stage = 0;
            phase ^= 1;
          }
        });
        tc_commit(tfull0 + 8 * acc);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: TMEM -> registers -> (smem -> TMA | global)
    const int quarter = warp & 3;              // TMEM lanes 32*quarter .. +31
    const int half = (warp - 4) >> 2;          // which half of the tile's columns
    uint8_t* buf = staging + (warp - 4) * bt.box_bytes;
    uint32_t box_seq = 0;   // staging-buffer alternation, continued across units
    const uint32_t ld_bar = smem_u32(bars + 2 * nst + 6 + 2 * (warp - 4));   // fused-epilogue input loads
    uint32_t ld_phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int u = blockIdx.x; u < num_units; u += gridDim.x) {
      const Unit x = decode_unit<BM, BN>(bt, u);
      const TcProblem& pr = bt.p[x.prob];
      mbar_wait(tfull0 + 8 * acc, acc_phase);
      tc_fence_after();
      if (bt.csplit > 1) {
        if constexpr (std::is_same<OutT, float>::value) {   // splits add into C in rank order
          const int rnk = static_cast<int>(cluster_rank());
          csplit_chain<BN>(pr, x, tmem_base + acc * BN, quarter, half, lane, x.m0 + quarter * 32, buf, box_seq,
                           smem_u32(bars + 2 * nst + 22 + (warp - 4)), rnk + 1 < bt.csplit ? rnk + 1 : -1);
        } else {
          // the partial goes to this CTA's shared memory (the pipeline stages
          // are idle: this was the CTA's only unit); the cluster reduces it
          // after the loop
          fence_async_smem();
          csplit_drain<BN>(tmem_base + acc * BN, quarter, half, lane, smem, x.kb0 >= x.kb1);
        }
      } else {
        epilogue_unit<BN, OutT>(pr, tmem_base + acc * BN, quarter, half, lane, x.m0 + quarter * 32, x.n0, x.split,
                                buf, box_seq, ld_bar, ld_phase, nullptr);
      }
      tc_fence_before();
      mbar_arrive(tempty0 + 8 * acc);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
    hap::pdl_trigger();   // last tile drained: let the next kernel start launching
    if (lane == 0) bulk_wait_all();
  }
  if (bt.csplit > 1 && !std::is_same<OutT, float>::value) {   // every thread of the cluster: both barriers
    cluster_sync_all();   // all partials are in shared memory
    if (warp >= 4 && static_cast<int>(blockIdx.x) < num_units) {
      const Unit x = decode_unit<BM, BN>(bt, blockIdx.x);
      csplit_finish<BN, OutT>(bt, bt.p[x.prob], x.prob, x.m0, x.n0, smem, static_cast<int>(cluster_rank()), bt.csplit,
                              threadIdx.x - 128);
    }
    cluster_sync_all();   // every peer has read this CTA's partial
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(G::kTmemCols));
  }
}

// ------------------------------------------------------------------ 2-CTA (SM pair) variant
// A cluster of two CTAs on one TPC computes a 256 x BN tile with
// tcgen05.mma.cta_group::2: CTA r stages rows [128r, 128r+128) of A and
// columns [r*BN/2, (r+1)*BN/2) of B; the pair's tensor cores read the peer's
// B half, so each SM moves half the B bytes of the single-CTA kernel.  CTA 0
// (the leader) issues every MMA; both CTAs' TMA loads complete on the
// leader's full barrier, the leader's commits multicast to both CTAs' empty
// and TMEM-full barriers, and both epilogues release the accumulator on the
// leader's TMEM-empty barrier.
// BN in {128, 192, 256}; each CTA stages BN/2 columns of B.  MN-major B is
// loaded in 64-column TMA boxes, so a 96-column half loads 128 columns (the
// MMA reads the first 96).
template <int BN, bool kBMN = false>
struct Cfg2 {
  static constexpr int kHalfLoaded = kBMN ? ((BN / 2 + 63) / 64) * 64 : BN / 2;
  static constexpr int kABytes = 128 * BK * 2;
  static constexpr int kBBytes = kHalfLoaded * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN <= 256 ? 256 : 512;
  static int smem(int nst, int box) { return nst * kStageBytes + kEpiWarps * box + 512 + 1024; }
};


__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_bar) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_cluster(uint32_t cluster_bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cluster.b64 _, [%0], %1;" ::"r"(cluster_bar),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred done;\n"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], %1;\n\t"
      "@!done bra WAITC_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t leader_bar,
                                                 int32_t x, int32_t y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tc_mma_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// Arrive on `bar` in both CTAs of the pair whose leader (even cluster rank)
// is `leader`.
__device__ __forceinline__ void tc_commit_pair(uint32_t bar, uint32_t leader) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(bar),
      "h"(static_cast<uint16_t>(3u << leader))
      : "memory");
}


template <int BN, bool kAMN, bool kBMN, typename OutT>
__global__ void __launch_bounds__(kThreads, 1) gemm_tc2_kernel(const __grid_constant__ TcBatch bt) {
  using G = Cfg2<BN, kBMN>;
  constexpr int HB = BN / 2;  // B columns of the tile each CTA supplies
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int nst = bt.nst;
  uint8_t* staging = smem + nst * G::kStageBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(staging + kEpiWarps * bt.box_bytes);
  const uint32_t full0 = smem_u32(bars);
  const uint32_t empty0 = smem_u32(bars + nst);
  const uint32_t tfull0 = smem_u32(bars + 2 * nst);
  const uint32_t tempty0 = smem_u32(bars + 2 * nst + 2);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * nst + 4);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // launched in clusters of 2 (one SM pair) or, under cluster split K, of
  // 2 x csplit (the pairs of one output tile): the pair is the CTAs whose
  // cluster ranks differ in bit 0, its leader the even one
  const uint32_t crank = cluster_rank();
  const uint32_t rank = crank & 1u;
  const uint32_t leader = crank & ~1u;
  const int pair = blockIdx.x >> 1;
  const int num_pairs = gridDim.x >> 1;
  if (threadIdx.x == 0) HAP_TRACE(0);

  if (warp == 0 && lane == 0) {
    for (int q = 0; q < bt.count; ++q) {
      tma_prefetch(&bt.p[q].a);
      tma_prefetch(&bt.p[q].b);
    }
  }
  if (warp == 3) warm_params(bt, lane);
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(full0 + 8 * s, 2);   // one producer arrival per CTA (+ both CTAs' bytes)
      mbar_init(empty0 + 8 * s, 1);  // the leader's multicast commit
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(tfull0 + 8 * a, 1);
      mbar_init(tempty0 + 8 * a, 2 * kEpiWarps);  // one arrival per epilogue warp of both CTAs
    }
    for (int w = 0; w < 2 * kEpiWarps; ++w) mbar_init(smem_u32(bars + 2 * nst + 6 + w), 1);
    for (int w = 0; w < kEpiWarps; ++w) mbar_init(smem_u32(bars + 2 * nst + 22 + w), 1);   // split-K turns
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(G::kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  hap::pdl_wait();   // everything above touched no global memory
  if (threadIdx.x == 0) HAP_TRACE(1);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs)
      int stage = 0;
      uint32_t phase = 0;
      unsigned long long w_empty = 0;
#ifdef HAP_GEMM_TRACE
      bool traced = false;
#endif
#ifdef HAP_GEMM_TRACE
      HAP_TRACE(29);
      bool traced_a = false, traced_b = false;
#endif
      PairCursor<BN> cur(bt, pair, num_pairs);
      Unit x;
      while (cur.next(bt, x)) {
        const int m0 = x.m0 + 128 * static_cast<int>(rank);
        const int n0 = x.n0 + HB * static_cast<int>(rank);
        for_each_kblock(bt, x, [&](int q, int kb) {
#ifdef HAP_GEMM_TRACE
          HAP_TRACE_ONCE(27, traced_a);
#endif
          HAP_TIMED(w_empty, mbar_wait_cluster(empty0 + 8 * stage, phase ^ 1));
          const uint32_t leader_full = map_to_cta(full0 + 8 * stage, leader);
          if (rank == 0) mbar_expect_tx_cluster(leader_full, 2 * G::kStageBytes);
          else mbar_arrive_cluster(leader_full);
#ifdef HAP_GEMM_TRACE
          HAP_TRACE_ONCE(28, traced_b);
#endif
          const uint32_t sa = smem_u32(smem + stage * G::kStageBytes);
          const uint32_t sb = sa + G::kABytes;
          const int k0 = kb * BK;
          const CUtensorMap* ma = &bt.p[q].a;
          const CUtensorMap* mb = &bt.p[q].b;
          if (kAMN) {
            tma_load_2d_pair(sa, ma, leader_full, m0, k0);
            tma_load_2d_pair(sa + BK * 128, ma, leader_full, m0 + 64, k0);
          } else {
            tma_load_2d_pair(sa, ma, leader_full, k0, m0);
          }
          if (kBMN) {
#pragma unroll
            for (int c = 0; c < G::kHalfLoaded / 64; ++c)
              tma_load_2d_pair(sb + c * BK * 128, mb, leader_full, n0 + 64 * c, k0);
          } else {
            tma_load_2d_pair(sb, mb, leader_full, k0, n0);
          }
#ifdef HAP_GEMM_TRACE
          HAP_TRACE_ONCE(2, traced);
          HAP_TRACE(9);
#endif
          if (++stage == nst) {
            stage = 0;
            phase ^= 1;
          }
        });
      }
#ifdef HAP_GEMM_TRACE
      trace_put(14, w_empty);
#endif
      (void)w_empty;
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (leader CTA only)
      constexpr uint32_t kIdesc = idesc(256, BN, kAMN, kBMN);
      constexpr uint32_t kALbo = kAMN ? BK * 128 : 16;
      constexpr uint32_t kBLbo = kBMN ? BK * 128 : 16;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      unsigned long long w_full = 0, w_tempty = 0;
#ifdef HAP_GEMM_TRACE
      bool traced = false;
#endif
      PairCursor<BN> cur(bt, pair, num_pairs);
      Unit x;
      while (cur.next(bt, x)) {
        HAP_TIMED(w_tempty, mbar_wait_cluster(tempty0 + 8 * acc, acc_phase ^ 1));
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        bool first = true;
        for_each_kblock(bt, x, [&](int, int) {
          HAP_TIMED(w_full, mbar_wait_cluster(full0 + 8 * stage, phase));
          tc_fence_after();
#ifdef HAP_GEMM_TRACE
          if (first) { HAP_TRACE_ONCE(3, traced); HAP_TRACE(10); }
#endif
          const uint32_t sa = smem_u32(smem + stage * G::kStageBytes);
          const uint32_t sb = sa + G::kABytes;
#pragma unroll
          for (int kk = 0; kk < BK / UMMA_K; ++kk) {
            const uint32_t aoff = kAMN ? kk * UMMA_K * 128 : kk * UMMA_K * 2;
            const uint32_t boff = kBMN ? kk * UMMA_K * 128 : kk * UMMA_K * 2;
            tc_mma_pair(d_tmem, sdesc(sa + aoff, kALbo, 1024), sdesc(sb + boff, kBLbo, 1024), kIdesc,
                        (!first) || (kk != 0));
          }
          first = false;
          tc_commit_pair(empty0 + 8 * stage, leader);
          if (++stage == nst) {
            stage = 0;
            phase ^= 1;
          }
        });
        tc_commit_pair(tfull0 + 8 * acc, leader);
        HAP_TRACE(4);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
#ifdef HAP_GEMM_TRACE
      trace_put(12, w_full);
      trace_put(13, w_tempty);
#endif
      (void)w_full;
      (void)w_tempty;
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs): own 128 rows of the 256-row tile
    const int quarter = warp & 3;
    const int half = (warp - 4) >> 2;
    uint8_t* buf = staging + (warp - 4) * bt.box_bytes;
    uint32_t box_seq = 0;   // staging-buffer alternation, continued across units
    const uint32_t ld_bar = smem_u32(bars + 2 * nst + 6 + 2 * (warp - 4));   // fused-epilogue input loads
    uint32_t ld_phase = 0;
    const uint32_t leader_tempty = map_to_cta(tempty0, leader);
    int acc = 0;
    uint32_t acc_phase = 0;
#ifdef HAP_GEMM_TRACE
    bool traced = false;
#endif
    PairCursor<BN> cur(bt, pair, num_pairs);
    Unit x;
    unsigned long long w_tfull = 0;
    while (cur.next(bt, x)) {
      const TcProblem& pr = bt.p[x.prob];
      const int m0 = x.m0 + 128 * static_cast<int>(rank);
      HAP_TIMED(w_tfull, mbar_wait_cluster(tfull0 + 8 * acc, acc_phase));
      tc_fence_after();
#ifdef HAP_GEMM_TRACE
      if (warp == 4 && lane == 0) { HAP_TRACE_ONCE(5, traced); HAP_TRACE(11); }
#endif
      if (bt.csplit > 1) {   // cluster split K
        if constexpr (std::is_same<OutT, float>::value) {   // the pairs add into C in rank order
          const int nxt = static_cast<int>(crank) + 2;
          csplit_chain<BN>(pr, x, tmem_base + acc * BN, quarter, half, lane, m0 + quarter * 32, buf, box_seq,
                           smem_u32(bars + 2 * nst + 22 + (warp - 4)), nxt < 2 * bt.csplit ? nxt : -1);
        } else {   // partial to this CTA's idle pipeline smem, reduced after the loop
          fence_async_smem();
          csplit_drain<BN>(tmem_base + acc * BN, quarter, half, lane, smem, x.kb0 >= x.kb1);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_tempty + 8 * acc);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
        continue;
      }
      // stream-K: this CTA's 128 x BN share of a cut tile's partial
      float* part = nullptr;
      unsigned* flag = nullptr;
      if (x.sk_kind) {
        part = bt.sk_ws + (static_cast<size_t>(x.sk_slot) * 2 + rank) * 128 * BN;
        flag = bt.sk_flags + (static_cast<size_t>(x.sk_slot) * 2 + rank) * kEpiWarps + (warp - 4);
      }
      if (x.sk_kind == 1) {
        write_partial<BN>(tmem_base + acc * BN, quarter, half, lane, part);
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release_gpu(flag, 1u);
      } else {
        if (x.sk_kind == 2) {
          if (lane == 0)
            while (ld_acquire_gpu(flag) == 0) __nanosleep(32);
          __syncwarp();
        }
        epilogue_unit<BN, OutT>(pr, tmem_base + acc * BN, quarter, half, lane, m0 + quarter * 32, x.n0, x.split,
                                buf, box_seq, ld_bar, ld_phase, x.sk_kind == 2 ? part : nullptr);
        if (x.sk_kind == 2 && lane == 0) *flag = 0u;   // consumed: ready for the next launch
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty + 8 * acc);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
#ifdef HAP_GEMM_TRACE
    if (warp == 4 && lane == 0) trace_put(15, w_tfull);
#endif
    (void)w_tfull;
    hap::pdl_trigger();   // last tile drained: let the next kernel start launching
    if (warp == 4 && lane == 0) HAP_TRACE(6);
    if (lane == 0) bulk_wait_all();
    if (warp == 4 && lane == 0) HAP_TRACE(7);
  }
  if (bt.csplit > 1 && !std::is_same<OutT, float>::value) {   // every thread of the cluster: both barriers
    cluster_sync_all();   // all partials are in shared memory
    if (warp >= 4 && pair < bt.total_units) {
      const Unit x = decode_unit<256, BN>(bt, pair);
      // CTAs holding the same 128 rows (same rank in their pairs) reduce together
      csplit_finish<BN, OutT>(bt, bt.p[x.prob], x.prob, x.m0 + 128 * static_cast<int>(rank), x.n0, smem,
                              static_cast<int>(crank >> 1), bt.csplit, threadIdx.x - 128, 2, static_cast<int>(rank));
    }
    cluster_sync_all();   // every peer has read this CTA's partial
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(G::kTmemCols));
  }
  if (threadIdx.x == 0) HAP_TRACE(8);
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 tensor map: `inner` contiguous elements per row, `outer` rows of
// pitch `ld` elements, box {64, box_outer}, 128B swizzle, zero OOB fill.
bool make_map(CUtensorMap* map, const void* ptr, int64_t inner, int64_t outer, int64_t ld,
              int box_outer) {
  ensure_context();
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_outer)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Output tensor map for the TMA epilogue: boxes of 128 bytes x 32 rows.
bool make_map_c(CUtensorMap* map, void* ptr, hap_dtype dt, int64_t inner, int64_t outer, int64_t ld, int bn,
                int box_w = 0) {
  ensure_context();
  auto fn = encode_fn();
  if (!fn) return false;
  const int es = dt == HAP_BF16 ? 2 : 4;
  const int wide = 128 / es;                               // must match drain_accumulator's W
  const int w = box_w ? box_w : (((bn / 2) % wide == 0) ? wide : wide / 2);
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * es};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(w), 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, dt == HAP_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ptr,
                  dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  w * es == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}


template <typename K>
hap_status launch_batch(K kern, int smem_bytes, const TcBatch& bt, int grid, cudaStream_t stream,
                        const char* what, int cluster = 0) {
  static_assert(sizeof(TcBatch) < 4096, "TcBatch must fit the kernel parameter space");
  // per-instantiation once: large dynamic shared memory
  static std::mutex mu;
  static std::vector<const void*> configured;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (std::find(configured.begin(), configured.end(), reinterpret_cast<const void*>(kern)) == configured.end()) {
      HAP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit));
      configured.push_back(reinterpret_cast<const void*>(kern));
    }
  }
  if (cluster > 1) {
    set_carveout(kern);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem_bytes;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled();
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = cluster;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaLaunchKernelEx(&cfg, kern, bt);
    return launch_status(what);
  }
  launch_k(kern, dim3(grid), dim3(kThreads), smem_bytes, stream, bt);
  return launch_status(what);
}

template <int BN, bool kAMN, bool kBMN, typename OutT>
hap_status launch_shape(bool pair, const TcBatch& bt_in, int cap, cudaStream_t stream) {
  TcBatch bt = bt_in;
  bool fused = false;
  for (int q = 0; q < bt.count; ++q) fused = fused || bt.p[q].epi != EPI_OP_NONE;
  bt.box_bytes = fused ? kEpiBoxBytesFused : kEpiBoxBytes;
  if (pair || BN == 192) {   // 192-wide tiles exist only for SM pairs
    using G = Cfg2<BN, kBMN>;
    bt.nst = stages_for(G::kStageBytes, bt.box_bytes);
    // clusters of one pair, or (cluster split K) of the csplit pairs of a tile, one unit each
    const int pairs = bt.csplit > 1 ? bt.total_units : std::min<int>(bt.total_units, std::max(1, cap / 2));
    return launch_batch(gemm_tc2_kernel<BN, kAMN, kBMN, OutT>, G::smem(bt.nst, bt.box_bytes), bt, 2 * pairs, stream,
                        "gemm_tc2_kernel", bt.csplit > 1 ? 2 * bt.csplit : 2);
  }
  if constexpr (BN != 192) {
    using G = Cfg<BN>;
    bt.nst = stages_for(G::kStageBytes, bt.box_bytes);
    const int smem = G::smem(bt.nst, bt.box_bytes);
    if (bt.csplit > 1)   // one CTA per unit, the splits of a tile one cluster
      return launch_batch(gemm_tc_kernel<BN, kAMN, kBMN, OutT>, smem, bt, bt.total_units, stream,
                          "gemm_tc_kernel (cluster split K)", bt.csplit);
    return launch_batch(gemm_tc_kernel<BN, kAMN, kBMN, OutT>, smem, bt, std::min(bt.total_units, cap),
                        stream, "gemm_tc_kernel");
  }
  return HAP_ERR_UNSUPPORTED;
}

template <typename OutT>
hap_status launch_dispatch(bool pair, int bn, bool amn, bool bmn, const TcBatch& bt, int cap, cudaStream_t s) {
#define HAP_TC_CASE(BNV, A, B) \
  if (bn == BNV && amn == A && bmn == B) return launch_shape<BNV, A, B, OutT>(pair, bt, cap, s);
  HAP_TC_CASE(256, false, false) HAP_TC_CASE(256, false, true) HAP_TC_CASE(256, true, false)
  HAP_TC_CASE(256, true, true) HAP_TC_CASE(128, false, false) HAP_TC_CASE(128, false, true)
  HAP_TC_CASE(128, true, false) HAP_TC_CASE(128, true, true) HAP_TC_CASE(192, false, false)
  HAP_TC_CASE(192, false, true) HAP_TC_CASE(192, true, false) HAP_TC_CASE(192, true, true)
#undef HAP_TC_CASE
  set_error("gemm: unsupported tile shape");
  return HAP_ERR_UNSUPPORTED;
}

// Tile shape of a batch: single-CTA 128 x BN or SM-pair 256 x BN
// (cta_group::2), BN in {128, 192, 256}, plus a split-K factor when the tiles
// alone cannot fill the SMs and the split's extra pass pays for itself.  Each
// candidate is scored by the fraction of the capped SMs kept busy across the
// persistent rounds, times a per-shape efficiency (operand bytes per MMA: the
// pair tile halves B traffic per SM; 128-wide tiles are smem-bandwidth bound).
struct Shape {
  int bn, splits, kb_per_split;
  bool pair;
  bool cl = false;   // split K over a thread-block cluster (single-CTA tiles, DSMEM reduction)
};

// Cluster split factors: S CTAs (single-CTA tiles) or S SM pairs (2S CTAs)
// per cluster, within the portable cluster size 8, the tile's 128 rows per
// CTA dividing evenly among the S.
inline bool cluster_split_ok(int64_t splits, bool pair) {
  return splits == 2 || splits == 4 || (splits == 8 && !pair);
}

Shape choose_shape(const int64_t* Ms, const int64_t* Ns, const int64_t* Ks, int count, int sum_k, bool allow_split,
                   bool fp32_out, int cap, int allow_pair) {
  // K blocks a unit walks: the concatenated K of a sum, else the largest
  // problem's (grouped problems with less K simply walk fewer blocks)
  int64_t k_blocks = 0;
  for (int q = 0; q < count; ++q) {
    const int64_t kb = (Ks[q] + BK - 1) / BK;
    k_blocks = sum_k ? k_blocks + kb : std::max(k_blocks, kb);
  }
  struct Cand { bool pair; int bn; double weight; };
  const Cand cands[] = {{true, 256, 1.0}, {true, 192, 0.85}, {true, 128, 0.8}, {false, 256, 0.75},
                        {false, 128, 0.65}};
  int64_t min_m = Ms[0];
  for (int q = 0; q < count; ++q) min_m = std::min(min_m, Ms[q]);
  // Best candidate without and with split-K, each by the fraction of the
  // capped SMs kept busy across the persistent rounds times the shape's
  // efficiency; est_us is a rough critical path (per-SM K-block time of a
  // BN-wide tile at full MMA rate / efficiency, times the K blocks each SM walks).
  struct Pick { Shape s; double score; double est_us; };
  Pick plain{{256, 1, static_cast<int>(k_blocks), false}, -1.0, 1e30};
  Pick split = plain;
  for (const Cand& c : cands) {
    if (c.pair && (!allow_pair || min_m < 256 || cap < 2)) continue;
    const int64_t rows = c.pair ? 256 : 128;
    const int64_t slots = c.pair ? cap / 2 : cap;
    int64_t tiles = 0;
    for (int q = 0; q < (sum_k ? 1 : count); ++q) tiles += ((Ms[q] + rows - 1) / rows) * ((Ns[q] + c.bn - 1) / c.bn);
    const double t_kb = 0.26 * c.bn / 256.0 / c.weight;
    for (int want_split = 0; want_split < 2; ++want_split) {
      int64_t splits = 1;
      if (want_split) {
        if (!allow_split || tiles >= slots || k_blocks < 8) continue;
        splits = std::max<int64_t>(1, std::min<int64_t>(slots / tiles, k_blocks / 4));
      }
      const int64_t kps = (k_blocks + splits - 1) / splits;
      splits = (k_blocks + kps - 1) / kps;
      if (want_split && splits < 2) continue;
      const int64_t work = tiles * splits;
      const int64_t rounds = (work + slots - 1) / slots;
      const double score = static_cast<double>(work) / static_cast<double>(rounds * slots) * c.weight;
      Pick& best = want_split ? split : plain;
      const double s_adj = want_split ? score * 0.97 : score;   // partial-sum traffic
      if (s_adj > best.score + 1e-9)
        best = {{c.bn, static_cast<int>(splits), static_cast<int>(kps), c.pair}, s_adj,
                static_cast<double>(rounds * kps) * t_kb};
    }
  }
  // Cluster split K (single-CTA tiles): the S splits of a tile reduce through
  // distributed shared memory inside the launch — a ~1 us tail.
  Pick cl = plain;
  cl.score = -1.0;
  if (allow_split && k_blocks >= 8) {
    for (const Cand& c : cands) {
      if (c.pair && (!allow_pair || min_m < 256 || cap < 4)) continue;
      const int64_t rows = c.pair ? 256 : 128;
      const int64_t slots = c.pair ? cap / 2 : cap;
      int64_t tiles = 0;
      for (int q = 0; q < (sum_k ? 1 : count); ++q) tiles += ((Ms[q] + rows - 1) / rows) * ((Ns[q] + c.bn - 1) / c.bn);
      const double t_kb = 0.26 * c.bn / 256.0 / c.weight;
      for (int64_t S = 2; S <= 8; S *= 2) {
        if (!cluster_split_ok(S, c.pair) || tiles * S > slots || k_blocks / S < 2) break;
        const int64_t kps = (k_blocks + S - 1) / S;
        if ((S - 1) * kps >= k_blocks) continue;   // every split walks at least one K block
        // fp32: the splits' adds into C run one after another (~0.7 us each);
        // bf16: the DSMEM reduction measured ~4 us beyond the K walk
        const double est = static_cast<double>(kps) * t_kb + (fp32_out ? 0.7 * static_cast<double>(S) : 4.0);
        if (cl.score < 0 || est < cl.est_us) {
          cl = {{c.bn, static_cast<int>(S), static_cast<int>(kps), c.pair}, 1.0, est};
          cl.s.cl = true;
        }
      }
    }
  }
  // Split K through the workspace stores fp32 partial slices and sums them in
  // order in a second launch (split_reduce_kernel): a serial tail (~5 us
  // measured on B200), so split only when the shortened K walk saves more.
  constexpr double kSplitTailUs = 5.0;
  double best_us = plain.score > 0 ? plain.est_us : 1e30;
  Shape best = plain.score > 0 ? plain.s : split.s;
  if (split.score > 0 && split.est_us + kSplitTailUs < best_us) {
    best_us = split.est_us + kSplitTailUs;
    best = split.s;
  }
  if (cl.score > 0 && cl.est_us < best_us) best = cl.s;
  return best;
}

// Every tile shape / split choose_shape considers (the autotuner times them).
void candidate_shapes(const int64_t* Ms, const int64_t* Ns, const int64_t* Ks, int count, int sum_k,
                      bool allow_split, int cap, int allow_pair, std::vector<Shape>& out) {
  int64_t k_blocks = 0;
  for (int q = 0; q < count; ++q) {
    const int64_t kb = (Ks[q] + BK - 1) / BK;
    k_blocks = sum_k ? k_blocks + kb : std::max(k_blocks, kb);
  }
  int64_t min_m = Ms[0];
  for (int q = 0; q < count; ++q) min_m = std::min(min_m, Ms[q]);
  const struct { bool pair; int bn; } cs[] = {{true, 256}, {true, 192}, {true, 128}, {false, 256}, {false, 128}};
  for (const auto& c : cs) {
    if (c.pair && (!allow_pair || min_m < 256 || cap < 2)) continue;
    const int64_t rows = c.pair ? 256 : 128;
    const int64_t slots = c.pair ? cap / 2 : cap;
    int64_t tiles = 0;
    for (int q = 0; q < (sum_k ? 1 : count); ++q) tiles += ((Ms[q] + rows - 1) / rows) * ((Ns[q] + c.bn - 1) / c.bn);
    out.push_back({c.bn, 1, static_cast<int>(k_blocks), c.pair});
    if (!allow_split || tiles >= slots || k_blocks < 8) continue;
    const int64_t top = std::max<int64_t>(1, std::min<int64_t>(slots / tiles, k_blocks / 4));
    for (int64_t want : {int64_t(2), top}) {
      if (want < 2 || want > top) continue;
      const int64_t kps = (k_blocks + want - 1) / want;
      const int64_t splits = (k_blocks + kps - 1) / kps;
      if (splits < 2) continue;
      Shape sh{c.bn, static_cast<int>(splits), static_cast<int>(kps), c.pair};
      bool dup = false;
      for (const Shape& o : out) dup = dup || (o.bn == sh.bn && o.pair == sh.pair && o.splits == sh.splits && !o.cl);
      if (!dup) out.push_back(sh);
    }
    for (int64_t S = 2; S <= 8; S *= 2) {   // cluster split K
      if (!cluster_split_ok(S, c.pair) || tiles * S > slots || k_blocks / S < 2) break;
      const int64_t kps = (k_blocks + S - 1) / S;
      if ((S - 1) * kps >= k_blocks) continue;
      Shape sh{c.bn, static_cast<int>(S), static_cast<int>(kps), c.pair};
      sh.cl = true;
      out.push_back(sh);
    }
  }
}

// C (+)= sum over s of ws[s] — the K splits' partial tiles added in split
// order (fixed, so repeated launches give identical bits).  A thread owns 4
// consecutive columns of a row; every split's load is issued before the sum.
//
// Split K under a residual epilogue (bf16 outputs): the reduction applies it
// with the fused path's roundings — HAP_EPI_ADD: C = bf16(sum + R);
// HAP_EPI_ADD2: C = bf16(sum), Y = bf16(bf16(sum) + R).  (ADD onto C itself
// is the plain accumulate.)
template <typename OutT>
__global__ void __launch_bounds__(256) split_reduce_kernel(const float* __restrict__ ws, int splits,
                                                           int64_t slice, int64_t ld, OutT* __restrict__ C,
                                                           int64_t ldc, int M, int N, int accumulate, int vec,
                                                           int epi, const __nv_bfloat16* __restrict__ R,
                                                           int64_t ldr, __nv_bfloat16* __restrict__ Y,
                                                           int64_t ldy) {
  hap::pdl_enter();
  const int64_t nq = (static_cast<int64_t>(N) + 3) / 4;
  const int64_t total = static_cast<int64_t>(M) * nq;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / nq;
    const int col = static_cast<int>(i - row * nq) * 4;
    const float* src = ws + row * ld + col;
    float4 acc = __ldcg(reinterpret_cast<const float4*>(src));
    constexpr int U = 8;
    for (int s0 = 1; s0 < splits; s0 += U) {
      float4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (s0 + u < splits) v[u] = __ldcg(reinterpret_cast<const float4*>(src + (s0 + u) * slice));
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (s0 + u < splits) {
          acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
        }
    }
    const float a[4] = {acc.x, acc.y, acc.z, acc.w};
    OutT* dst = C + row * ldc + col;
    if (vec && col + 4 <= N) {
      if constexpr (std::is_same<OutT, float>::value) {
        float4 o = make_float4(a[0], a[1], a[2], a[3]);
        if (accumulate) {
          const float4 c = *reinterpret_cast<const float4*>(dst);
          o.x += c.x; o.y += c.y; o.z += c.z; o.w += c.w;
        }
        *reinterpret_cast<float4*>(dst) = o;
      } else {
        auto ld4 = [](const void* p, float (&f)[4]) {
          const uint2 c = *reinterpret_cast<const uint2*>(p);
          const float2 lo = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&c.x));
          const float2 hi = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&c.y));
          f[0] = lo.x; f[1] = lo.y; f[2] = hi.x; f[3] = hi.y;
        };
        auto st4 = [](void* p, const float (&f)[4]) {
          __nv_bfloat162 lo = __floats2bfloat162_rn(f[0], f[1]), hi = __floats2bfloat162_rn(f[2], f[3]);
          uint2 o;
          o.x = *reinterpret_cast<uint32_t*>(&lo);
          o.y = *reinterpret_cast<uint32_t*>(&hi);
          *reinterpret_cast<uint2*>(p) = o;
        };
        float f[4] = {a[0], a[1], a[2], a[3]}, x[4];
        if (accumulate) {
          ld4(dst, x);
#pragma unroll
          for (int e = 0; e < 4; ++e) f[e] += x[e];
        }
        if (epi != EPI_OP_NONE) ld4(R + row * ldr + col, x);
        if (epi == EPI_OP_ADD) {
#pragma unroll
          for (int e = 0; e < 4; ++e) f[e] += x[e];
        }
        st4(dst, f);
        if (epi == EPI_OP_ADD2) {
          float y[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) y[e] = bf16_round(f[e]) + x[e];
          st4(Y + row * ldy + col, y);
        }
      }
    } else {
      for (int e = 0; e < 4 && col + e < N; ++e) {
        float v = a[e];
        if (accumulate) v += to_f32(dst[e]);
        const float r = epi != EPI_OP_NONE ? to_f32(R[row * ldr + col + e]) : 0.f;
        if (epi == EPI_OP_ADD) v += r;
        dst[e] = from_f32<OutT>(v);
        if (epi == EPI_OP_ADD2) Y[row * ldy + col + e] = from_f32<__nv_bfloat16>(bf16_round(v) + r);
      }
    }
  }
}

}  // namespace tc

// ------------------------------------------------------------------ SIMT path
namespace simt {

constexpr int TM = 64, TN = 64, TK = 16;

template <typename Tin, typename Tout>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const Tin* __restrict__ A, int64_t lda,
                                                        int transA, const Tin* __restrict__ B,
                                                        int64_t ldb, int transB,
                                                        Tout* __restrict__ C, int64_t ldc,
                                                        int64_t M, int64_t N, int64_t K,
                                                        int accumulate) {
  hap::pdl_enter();
  __shared__ float As[TK][TM + 1];
  __shared__ float Bs[TK][TN + 1];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int64_t tiles_n = (N + TN - 1) / TN;
  const int64_t tiles = ((M + TM - 1) / TM) * tiles_n;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int64_t m0 = (t / tiles_n) * TM, n0 = (t % tiles_n) * TN;
    float acc[4][4] = {};
    for (int64_t k0 = 0; k0 < K; k0 += TK) {
      for (int i = threadIdx.x; i < TK * TM; i += 256) {
        const int kk = transA ? i / TM : i % TK;
        const int mm = transA ? i % TM : i / TK;
        const int64_t gm = m0 + mm, gk = k0 + kk;
        float v = 0.f;
        if (gm < M && gk < K) v = to_f32(transA ? A[gk * lda + gm] : A[gm * lda + gk]);
        As[kk][mm] = v;
      }
      for (int i = threadIdx.x; i < TK * TN; i += 256) {
        const int kk = transB ? i % TK : i / TN;
        const int nn = transB ? i / TK : i % TN;
        const int64_t gn = n0 + nn, gk = k0 + kk;
        float v = 0.f;
        if (gn < N && gk < K) v = to_f32(transB ? B[gn * ldb + gk] : B[gk * ldb + gn]);
        Bs[kk][nn] = v;
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < TK; ++kk) {
        float a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
        for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int64_t gm = m0 + ty * 4 + i;
      if (gm >= M) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t gn = n0 + tx * 4 + j;
        if (gn >= N) continue;
        float v = acc[i][j];
        if (accumulate) v += to_f32(C[gm * ldc + gn]);
        C[gm * ldc + gn] = from_f32<Tout>(v);
      }
    }
  }
}

}  // namespace simt

namespace {

int tma_epilogue() {
  static int mode = [] {
    const char* v = getenv("HAP_GEMM_TMA_EPI");
    return v ? atoi(v) : 1;
  }();
  return mode;
}

// HAP_GEMM_SPLIT=0 disables split-K.
int split_enabled() {
  static int mode = [] {
    const char* v = getenv("HAP_GEMM_SPLIT");
    return v ? atoi(v) : 1;
  }();
  return mode;
}

// HAP_GEMM_SK=1 enables stream-K (read per call, so tests can toggle it).
// Off by default: measured on the bench shapes (profiles/r01f_stream_k.md) the
// cut tiles' partial write + read costs more than the idle pairs it fills.
int sk_enabled() {
  const char* v = getenv("HAP_GEMM_SK");
  return v ? atoi(v) : 0;
}

int pair_mode() {
  static int mode = [] {
    const char* v = getenv("HAP_GEMM_PAIR");
    return v ? atoi(v) : 1;
  }();
  return mode;
}

bool tc_eligible(const void* A, int64_t lda, int transA, const void* B, int64_t ldb, int transB,
                 int64_t M, int64_t N, int64_t K, hap_dtype in_dtype) {
  if (in_dtype != HAP_BF16) return false;
  if (M <= 0 || N <= 0 || K <= 0) return false;
  if (M > (1LL << 31) - 1 || N > (1LL << 31) - 1 || K > (1LL << 31) - 1) return false;
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(B) & 15)) return false;
  if ((lda % 8) || (ldb % 8)) return false;
  // TMA needs the contiguous extent to cover at least one 16-byte chunk.
  const int64_t a_inner = transA ? M : K, b_inner = transB ? K : N;
  if (a_inner < 8 || b_inner < 8) return false;
  (void)transB;
  return tc::encode_fn() != nullptr;
}

template <typename Tin, typename Tout>
hap_status simt_launch(const void* A, int64_t lda, int transA, const void* B, int64_t ldb,
                       int transB, void* C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                       int accumulate, int sm_cap, cudaStream_t stream) {
  const int64_t tiles = ((M + simt::TM - 1) / simt::TM) * ((N + simt::TN - 1) / simt::TN);
  const int grid = capped_grid(tiles, sm_cap > 0 ? sm_cap * 4 : sm_count() * 4);
  hap::launch_k(simt::gemm_simt_kernel<Tin, Tout>, dim3(grid), dim3(256), 0, stream, 
      static_cast<const Tin*>(A), lda, transA, static_cast<const Tin*>(B), ldb, transB,
      static_cast<Tout*>(C), ldc, M, N, K, accumulate);
  return launch_status("gemm_simt_kernel");
}

}  // namespace
}  // namespace hap

using namespace hap;

extern "C" int hap_matmul_engine(const void* A, int64_t lda, int transA, const void* B,
                                 int64_t ldb, int transB, int64_t M, int64_t N, int64_t K,
                                 hap_dtype in_dtype) {
  return tc_eligible(A, lda, transA, B, ldb, transB, M, N, K, in_dtype) ? HAP_GEMM_TCGEN05
                                                                         : HAP_GEMM_SIMT;
}

namespace {

// Stream-K partial tiles and flags, one set per stream (launches on a stream
// are ordered; every flag is reset by the pair that consumes it).  Sized for
// the largest grid (74 SM pairs + 1 slot, 256-wide tiles); allocated outside
// stream capture only.
bool sk_workspace(cudaStream_t stream, float** ws, unsigned** flags) {
  const size_t slots = 148 / 2 + 1;
  void* w = nullptr;
  void* f = nullptr;
  if (!stream_scratch(stream, kScratchStreamK, slots * 2 * 128 * 256 * sizeof(float), false, &w) ||
      !stream_scratch(stream, kScratchStreamKFlags, slots * 2 * tc::kEpiWarps * sizeof(unsigned), true, &f))
    return false;
  *ws = static_cast<float*>(w);
  *flags = static_cast<unsigned*>(f);
  return true;
}

inline int64_t ws_pitch(int64_t n) { return (n + 3) / 4 * 4; }   // 16-byte rows for the TMA map

// Autotuned shapes (hap_matmul_tune), keyed by everything that decides the
// shape: problem extents, orientation, epilogue, output type, SM cap.
std::mutex& tune_mutex() {
  static std::mutex mu;
  return mu;
}
std::unordered_map<std::string, tc::Shape>& tune_cache() {
  static std::unordered_map<std::string, tc::Shape> cache;
  return cache;
}
std::string tune_key(const hap_gemm_desc* d, int count, int sum_k, bool fp32, int cap) {
  std::string k = std::to_string(count) + "/" + std::to_string(sum_k) + "/" + (fp32 ? "f" : "b") + "/" +
                  std::to_string(cap);
  for (int q = 0; q < count; ++q) {
    const hap_gemm_desc& g = d[q];
    k += "|" + std::to_string(g.M) + "x" + std::to_string(g.N) + "x" + std::to_string(g.K) + ":" +
         std::to_string(g.transA) + std::to_string(g.transB) + ":" + std::to_string(g.epi) + ":" +
         std::to_string(g.accumulate) + ":" + std::to_string(g.lda) + "," + std::to_string(g.ldb) + "," +
         std::to_string(g.ldc);
  }
  return k;
}

// Split K is allowed when every output's epilogue is plain or a residual add
// (the split reduction applies ADD / ADD2); the swish chains need the whole
// accumulator tile in the GEMM's epilogue.
bool split_fusable(const hap_gemm_desc* d, int nout) {
  for (int q = 0; q < nout; ++q)
    if (d[q].epi != HAP_EPI_NONE && d[q].epi != HAP_EPI_ADD && d[q].epi != HAP_EPI_ADD2) return false;
  return true;
}

// Build and launch one tcgen05 batch (all problems tc-eligible, same
// orientation, <= kMaxProblems).  sum_k: every problem adds into problem 0's
// output (same C, M, N), accumulate taken from problem 0.
hap_status tc_batch(const hap_gemm_desc* d, int count, int sum_k, hap_dtype out_dtype, int sm_cap,
                    cudaStream_t stream, const tc::Shape* force = nullptr) {
  const int cap = sm_cap > 0 && sm_cap < sm_count() ? sm_cap : sm_count();
  int64_t Ms[tc::kMaxProblems], Ns[tc::kMaxProblems], Ks[tc::kMaxProblems];
  for (int q = 0; q < count; ++q) {
    Ms[q] = d[q].M;
    Ns[q] = d[q].N;
    Ks[q] = d[q].K;
  }
  const bool fp32 = out_dtype == HAP_F32;
  const int nout = sum_k ? 1 : count;
  bool fused = false;
  for (int q = 0; q < nout; ++q) fused = fused || d[q].epi != HAP_EPI_NONE;
  HAP_CHECK_ARG(!fused || !fp32, "hap_matmul: fused epilogues need a bf16 output");
  // a fused epilogue runs once per output tile; under split K the residual
  // adds (ADD / ADD2) move into the split finish, the swish chains do not
  // split
  const bool may_split = split_enabled() != 0 && split_fusable(d, nout);
  tc::Shape shp = tc::choose_shape(Ms, Ns, Ks, count, sum_k, may_split, fp32, cap, pair_mode());
  if (force) {
    shp = *force;
  } else {
    std::lock_guard<std::mutex> lock(tune_mutex());
    auto it = tune_cache().find(tune_key(d, count, sum_k, fp32, cap));
    if (it != tune_cache().end()) shp = it->second;
  }
  auto problem_splits = [&](int q, const tc::Shape& sh) -> int64_t {
    if (sum_k) return sh.splits;
    const int64_t kb = (Ks[q] + tc::BK - 1) / tc::BK;
    const int64_t kps = std::max<int64_t>(1, std::min<int64_t>(sh.kb_per_split, kb));
    return (kb + kps - 1) / kps;
  };
  auto tiles_of = [&](int q, const tc::Shape& sh) -> int64_t {
    const int64_t r = sh.pair ? 256 : tc::BM;
    return ((Ms[q] + r - 1) / r) * ((Ns[q] + sh.bn - 1) / sh.bn);
  };
  // split-K partial slices: splits x (M rounded up to whole tiles) x pitch(N)
  // fp32 per output, in the stream's workspace
  float* ws = nullptr;
  auto slice_rows = [&](int q, const tc::Shape& sh) {
    const int64_t r = sh.pair ? 256 : tc::BM;
    return (Ms[q] + r - 1) / r * r;
  };
  const bool csplit = shp.cl && shp.splits > 1 && tc::cluster_split_ok(shp.splits, shp.pair);
  if (shp.cl && !csplit) shp = tc::choose_shape(Ms, Ns, Ks, count, sum_k, false, fp32, cap, pair_mode());
  if (shp.splits > 1 && !csplit) {
    int64_t need = 0;
    for (int q = 0; q < nout; ++q) {
      const int64_t sp = problem_splits(q, shp);
      if (sp > 1) need += sp * slice_rows(q, shp) * ws_pitch(Ns[q]);
    }
    void* w = nullptr;
    // no silent fallback: a different split factor would round differently
    HAP_CHECK_ARG(stream_scratch(stream, kScratchSplitWs, need * sizeof(float), false, &w),
                  "hap_matmul: no split-K workspace on this stream (out of memory, or its first split launch "
                  "is inside a CUDA graph capture: launch once eagerly first)");
    ws = static_cast<float*>(w);
  }
  const int rows = shp.pair ? 256 : tc::BM;
  const int b_box = shp.pair ? shp.bn / 2 : shp.bn;
  const bool amn = d[0].transA != 0, bmn = d[0].transB == 0;
  const size_t osz = dtype_size(out_dtype);
  tc::TcBatch bt;
  std::memset(&bt, 0, sizeof(bt));
  bt.count = count;
  bt.sum_k = sum_k;
  for (int q = 0; q < count; ++q) bt.sum_kb += static_cast<int>((d[q].K + tc::BK - 1) / tc::BK);
  int units = 0;
  int64_t ws_used = 0;
  struct SplitEpi { int epi; const void* R; int64_t ldr; void* Y; int64_t ldy; int vec; };
  SplitEpi sepi[tc::kMaxProblems] = {};
  for (int q = 0; q < count; ++q) {
    tc::TcProblem& pr = bt.p[q];
    const hap_gemm_desc& g = d[q];
    bool ok = g.transA ? tc::make_map(&pr.a, g.A, g.M, g.K, g.lda, tc::BK) : tc::make_map(&pr.a, g.A, g.K, g.M, g.lda, tc::BM);
    ok = ok && (g.transB ? tc::make_map(&pr.b, g.B, g.K, g.N, g.ldb, b_box) : tc::make_map(&pr.b, g.B, g.N, g.K, g.ldb, tc::BK));
    HAP_CHECK_ARG(ok, "hap_matmul: cuTensorMapEncodeTiled rejected the operand layout (problem " + std::to_string(q) +
                          " of " + std::to_string(count) + ": M " + std::to_string(g.M) + " N " + std::to_string(g.N) +
                          " K " + std::to_string(g.K) + " lda " + std::to_string(g.lda) + " ldb " +
                          std::to_string(g.ldb) + " trans " + std::to_string(g.transA) + std::to_string(g.transB) +
                          " A%16 " + std::to_string(reinterpret_cast<uintptr_t>(g.A) & 15) + " B%16 " +
                          std::to_string(reinterpret_cast<uintptr_t>(g.B) & 15) + " box " + std::to_string(b_box) +
                          (shp.pair ? " pair" : " cta") + ")");
    const hap_gemm_desc& out = sum_k ? d[0] : g;
    pr.C = out.C;
    pr.ldc = out.ldc;
    pr.M = static_cast<int>(out.M);
    pr.N = static_cast<int>(out.N);
    pr.K = static_cast<int>(g.K);
    pr.m_tiles = static_cast<int>((out.M + rows - 1) / rows);
    pr.n_tiles = static_cast<int>((out.N + shp.bn - 1) / shp.bn);
    pr.k_blocks = static_cast<int>((g.K + tc::BK - 1) / tc::BK);
    // grouped problems split K by the same factor (problems with fewer K
    // blocks get fewer splits); a sum splits its concatenated K blocks
    pr.splits = csplit ? 1 : static_cast<int>(problem_splits(q, shp));
    pr.kb_per_split = sum_k ? shp.kb_per_split : std::max(1, std::min(shp.kb_per_split, pr.k_blocks));
    if (pr.splits <= 1) {
      pr.splits = 1;
      pr.kb_per_split = sum_k ? bt.sum_kb : pr.k_blocks;
    }
    pr.accumulate = out.accumulate;
    pr.vec_ok = ((reinterpret_cast<uintptr_t>(out.C) & 15) == 0) && ((out.ldc * osz) % 16 == 0);
    // Epilogue: TMA bulk store when the output rows are 16-byte pitched; fp32
    // accumulation uses TMA reduce-add (one writer per element: in order); a
    // bf16 accumulate (read-modify-round) is the fused ADD of C itself; split
    // K stores fp32 partial slices, summed in order by split_reduce_kernel.
    pr.epi_mode = tc::EPI_DIRECT;
    pr.epi = (!sum_k || q == 0) ? out.epi : HAP_EPI_NONE;
    pr.epi_tag = out.epi_tag;
    int epi = pr.epi;
    const void* R = out.R;
    int64_t ldr = out.ldr;
    // K split (workspace slices or cluster): the reduction adds C itself when accumulating
    const bool splitting = csplit || pr.splits > 1;
    if (epi == HAP_EPI_NONE && !fp32 && out.accumulate && !splitting && pr.vec_ok && tma_epilogue()) {
      epi = HAP_EPI_ADD;
      R = out.C;
      ldr = out.ldc;
    }
    if (epi == HAP_EPI_ADD && out.accumulate && splitting) epi = HAP_EPI_NONE;   // += C: the accumulate
    pr.epi = epi;
    if (csplit && (!sum_k || q == 0)) {
      // cluster split K: the DSMEM finish applies accumulate and the residual
      // epilogue (split_fusable)
      HAP_CHECK_ARG(epi == HAP_EPI_NONE || epi == HAP_EPI_ADD || epi == HAP_EPI_ADD2,
                    "hap_matmul: this fused epilogue cannot split K");
      HAP_CHECK_ARG(epi == HAP_EPI_NONE || (R != nullptr && (epi != HAP_EPI_ADD2 || out.Y != nullptr)),
                    "hap_matmul: fused epilogue tensor R / Y is null");
      bt.fin_epi[q] = epi;
      bt.fin_R[q] = R;
      bt.fin_ldr[q] = ldr;
      bt.fin_Y[q] = out.Y;
      bt.fin_ldy[q] = out.ldy;
      pr.epi = HAP_EPI_NONE;
      pr.epi_mode = tc::EPI_DIRECT;
      // fp32: the split chain adds by TMA reduce-add when C is 16-byte pitched
      if (fp32 && pr.vec_ok && tma_epilogue() && tc::make_map_c(&pr.c, out.C, out_dtype, out.N, out.M, out.ldc, shp.bn))
        pr.epi_mode = tc::EPI_TMA_ADD;
    } else if (pr.splits > 1 && (!sum_k || q == 0)) {
      // split K: the ordered reduction applies the residual epilogue (split_fusable)
      HAP_CHECK_ARG(epi == HAP_EPI_NONE || epi == HAP_EPI_ADD || epi == HAP_EPI_ADD2,
                    "hap_matmul: this fused epilogue cannot split K");
      HAP_CHECK_ARG(epi == HAP_EPI_NONE || (R != nullptr && (epi != HAP_EPI_ADD2 || out.Y != nullptr)),
                    "hap_matmul: fused epilogue tensor R / Y is null");
      auto al8 = [](const void* ptr, int64_t ld) { return (reinterpret_cast<uintptr_t>(ptr) & 7) == 0 && ld % 4 == 0; };
      sepi[q] = {epi, R, ldr, out.Y, out.ldy, al8(R, ldr) && (epi != HAP_EPI_ADD2 || al8(out.Y, out.ldy))};
      pr.epi = HAP_EPI_NONE;
      pr.ws = ws + ws_used;
      pr.ws_ld = ws_pitch(out.N);
      pr.ws_rows = static_cast<int>(slice_rows(q, shp));
      ws_used += static_cast<int64_t>(pr.splits) * pr.ws_rows * pr.ws_ld;
      HAP_CHECK_ARG(tc::make_map_c(&pr.c, pr.ws, HAP_F32, out.N, static_cast<int64_t>(pr.splits) * pr.ws_rows,
                                   pr.ws_ld, shp.bn),
                    "hap_matmul: workspace tensor map rejected");
      pr.epi_mode = tc::EPI_SPLIT_WS;
    } else if (pr.epi != HAP_EPI_NONE) {
      HAP_CHECK_ARG(pr.vec_ok && tma_epilogue(),
                    "hap_matmul: fused epilogue needs a 16-byte pitched output and the TMA epilogue");
      HAP_CHECK_ARG(epi >= HAP_EPI_ADD && epi <= HAP_EPI_SWISH_BWD, "hap_matmul: unknown epilogue op");
      if (epi == HAP_EPI_ADD && out.accumulate) {
        HAP_CHECK_ARG(R == nullptr || R == out.C,
                      "hap_matmul: HAP_EPI_ADD with accumulate adds C itself (R must be C or null)");
        R = out.C;
        ldr = out.ldc;
      }
      HAP_CHECK_ARG(epi != HAP_EPI_SWISH_BWD || !out.accumulate,
                    "hap_matmul: the fused swish adjoint writes C (no accumulate)");
      auto map = [&](CUtensorMap* m, const void* ptr, int64_t ld, const char* what) -> bool {
        if (ptr == nullptr ||
            !tc::make_map_c(m, const_cast<void*>(ptr), HAP_BF16, out.N, out.M, ld, shp.bn, tc::kFusedW)) {
          set_error(std::string("hap_matmul: fused epilogue tensor ") + what +
                    " is null or not 16-byte aligned / pitched");
          return false;
        }
        return true;
      };
      bool ok = map(&pr.c, out.C, out.ldc, "C");
      if (epi == HAP_EPI_ADD) ok = ok && map(&pr.e1, R, ldr, "R");
      if (epi == HAP_EPI_ADD2) ok = ok && map(&pr.e1, R, ldr, "R") && map(&pr.e2, out.Y, out.ldy, "Y");
      if (epi == HAP_EPI_SWISH) ok = ok && map(&pr.e1, out.Y, out.ldy, "Y") && map(&pr.e2, out.Z, out.ldz, "Z");
      if (epi == HAP_EPI_SWISH_BWD) ok = ok && map(&pr.e1, R, ldr, "R") && map(&pr.e2, out.R2, out.ldr2, "R2");
      if (!ok) return HAP_ERR_ARG;
      pr.accumulate = 0;
      pr.epi_mode = tc::EPI_TMA_STORE;
    } else if (pr.vec_ok && tma_epilogue() && (!pr.accumulate || fp32) &&
               tc::make_map_c(&pr.c, out.C, out_dtype, out.N, out.M, out.ldc, shp.bn)) {
      pr.epi_mode = (fp32 && pr.accumulate) ? tc::EPI_TMA_ADD : tc::EPI_TMA_STORE;
    }
    pr.unit_begin = units;
    if (!sum_k || q == 0) units += pr.m_tiles * pr.n_tiles * pr.splits;
  }
  bt.total_units = units;
  if (csplit) {
    bt.csplit = shp.splits;
    bt.total_units = units * shp.splits;
  }
  // stream-K: one problem on SM pairs whose data-parallel rounds would leave
  // pairs idle (tile counts are products of 2s and 3s, the pair count 74 is
  // 2 x 37: the last round is rarely full).  Every pair gets the same number
  // of K-block iterations; needs at least one whole tile per pair.
  if (count == 1 && !sum_k && shp.pair && bt.p[0].splits == 1 && bt.p[0].epi_mode == tc::EPI_TMA_STORE &&
      sk_enabled()) {
    const int P = std::max(1, cap / 2);
    const int64_t T = static_cast<int64_t>(bt.p[0].m_tiles) * bt.p[0].n_tiles;
    const int64_t rounds = (T + P - 1) / P;
    const double eff = static_cast<double>(T) / static_cast<double>(rounds * P);
    float* skws = nullptr;
    unsigned* skflags = nullptr;
    // long tiles only: every cut costs an extra partial write / read and epilogue
    if (T >= P && eff < 0.93 && bt.p[0].k_blocks >= 16 && sk_workspace(stream, &skws, &skflags)) {
      bt.sk = 1;
      bt.sk_kb = bt.p[0].k_blocks;
      bt.sk_pairs = P;
      bt.sk_iters = T * bt.p[0].k_blocks;
      bt.sk_ws = skws;
      bt.sk_flags = skflags;
      bt.total_units = P;
    }
  }
  static const bool log_shapes = getenv("HAP_GEMM_LOG") != nullptr;
  if (log_shapes) {
    fprintf(stderr, "[hap gemm] count %d sum_k %d out %s cap %d -> %s BN %d splits %d%s kbps %d units %d sk %d |",
            count, sum_k, fp32 ? "f32" : "bf16", cap, shp.pair ? "pair" : "cta", shp.bn, shp.splits,
            csplit ? " (cluster)" : "", shp.kb_per_split, units, bt.sk);
    for (int q = 0; q < count; ++q)
      fprintf(stderr, " %lldx%lldx%lld t%d%d epi%d acc%d", static_cast<long long>(d[q].M),
              static_cast<long long>(d[q].N), static_cast<long long>(d[q].K), d[q].transA, d[q].transB, d[q].epi,
              d[q].accumulate);
    fprintf(stderr, "\n");
  }
  hap_status st = fp32 ? tc::launch_dispatch<float>(shp.pair, shp.bn, amn, bmn, bt, cap, stream)
                       : tc::launch_dispatch<__nv_bfloat16>(shp.pair, shp.bn, amn, bmn, bt, cap, stream);
  if (st != HAP_OK || csplit) return st;
  if (st != HAP_OK) return st;
  for (int q = 0; q < nout; ++q) {
    const tc::TcProblem& pr = bt.p[q];
    if (pr.epi_mode != tc::EPI_SPLIT_WS) continue;
    const int64_t work = static_cast<int64_t>(pr.M) * ((pr.N + 3) / 4);
    const int grid = capped_grid((work + 255) / 256, cap * 4);
    const int64_t slice = static_cast<int64_t>(pr.ws_rows) * pr.ws_ld;
    const SplitEpi& se = sepi[q];
    if (fp32)
      launch_k(tc::split_reduce_kernel<float>, dim3(grid), dim3(256), 0, stream, static_cast<const float*>(pr.ws),
               pr.splits, slice, pr.ws_ld, static_cast<float*>(pr.C), pr.ldc, pr.M, pr.N, pr.accumulate,
               pr.vec_ok, 0, nullptr, 0, nullptr, 0);
    else
      launch_k(tc::split_reduce_kernel<__nv_bfloat16>, dim3(grid), dim3(256), 0, stream,
               static_cast<const float*>(pr.ws), pr.splits, slice, pr.ws_ld, static_cast<__nv_bfloat16*>(pr.C),
               pr.ldc, pr.M, pr.N, pr.accumulate, pr.vec_ok && (se.epi == HAP_EPI_NONE || se.vec), se.epi,
               static_cast<const __nv_bfloat16*>(se.R), se.ldr, static_cast<__nv_bfloat16*>(se.Y), se.ldy);
    st = launch_status("split_reduce_kernel");
    if (st != HAP_OK) return st;
  }
  return HAP_OK;
}

hap_status simt_one(const hap_gemm_desc& g, hap_dtype in_dtype, hap_dtype out_dtype, int sm_cap,
                    cudaStream_t stream) {
  return HAP_DISPATCH_IO(in_dtype, out_dtype, [&] {
    return simt_launch<Tin, Tout>(g.A, g.lda, g.transA, g.B, g.ldb, g.transB, g.C, g.ldc, g.M, g.N, g.K,
                                  g.accumulate, sm_cap, stream);
  });
}

// Degenerate extents: M or N zero -> nothing; K zero -> C = 0 (or unchanged).
bool degenerate(const hap_gemm_desc& g, hap_dtype out_dtype, cudaStream_t stream, hap_status* st) {
  if (g.M == 0 || g.N == 0) {
    *st = HAP_OK;
    return true;
  }
  if (g.K == 0) {
    *st = HAP_OK;
    if (!g.accumulate) {
      const size_t osz = dtype_size(out_dtype);
      if (cudaMemset2DAsync(g.C, g.ldc * osz, 0, g.N * osz, g.M, stream) != cudaSuccess) {
        set_error("hap_matmul: cudaMemset2DAsync failed");
        *st = HAP_ERR_CUDA;
      }
    }
    return true;
  }
  return false;
}

}  // namespace

// Time every candidate tile shape / split of this batch on `stream` (outputs
// redirected to scratch buffers, inputs only read) and remember the fastest
// for later launches of the same signature.  Not during stream capture.
extern "C" hap_status hap_matmul_tune(const hap_gemm_desc* descs, int count, int sum_k, hap_dtype in_dtype,
                                      hap_dtype out_dtype, int sm_cap, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  HAP_CHECK_ARG(descs && count >= 0, "hap_matmul_tune: bad arguments");
  if (count == 0 || count > tc::kMaxProblems) return HAP_OK;
  for (int q = 0; q < count; ++q) {
    const hap_gemm_desc& g = descs[q];
    if (!(g.M > 0 && g.N > 0 && g.K > 0 && g.transA == descs[0].transA && g.transB == descs[0].transB &&
          tc_eligible(g.A, g.lda, g.transA, g.B, g.ldb, g.transB, g.M, g.N, g.K, in_dtype)))
      return HAP_OK;   // runs on the SIMT path or one by one: nothing to tune
  }
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  HAP_CUDA_TRY(cudaStreamIsCapturing(stream, &cs));
  HAP_CHECK_ARG(cs == cudaStreamCaptureStatusNone, "hap_matmul_tune: not during stream capture");
  const int cap = sm_cap > 0 && sm_cap < sm_count() ? sm_cap : sm_count();
  const bool fp32 = out_dtype == HAP_F32;
  {   // a signature is timed once per process (or imported): later executors reuse the choice
    std::lock_guard<std::mutex> lock(tune_mutex());
    if (tune_cache().count(tune_key(descs, count, sum_k, fp32, cap))) return HAP_OK;
  }
  const int nout = sum_k ? 1 : count;
  bool fused = false;
  for (int q = 0; q < nout; ++q) fused = fused || descs[q].epi != HAP_EPI_NONE;
  int64_t Ms[tc::kMaxProblems], Ns[tc::kMaxProblems], Ks[tc::kMaxProblems];
  for (int q = 0; q < count; ++q) {
    Ms[q] = descs[q].M;
    Ns[q] = descs[q].N;
    Ks[q] = descs[q].K;
  }
  std::vector<tc::Shape> cands;
  tc::candidate_shapes(Ms, Ns, Ks, count, sum_k, split_enabled() != 0 && split_fusable(descs, nout), cap,
                       pair_mode(), cands);
  if (cands.size() < 2) return HAP_OK;
  // scratch outputs: every written tensor of the batch
  const size_t osz = dtype_size(out_dtype);
  std::vector<void*> scratch;
  hap_gemm_desc t[tc::kMaxProblems];
  auto scratch_like = [&](int64_t rows, int64_t ld, size_t es) -> void* {
    void* p = nullptr;
    if (cudaMalloc(&p, static_cast<size_t>(rows) * ld * es) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    scratch.push_back(p);
    return p;
  };
  bool ok = true;
  for (int q = 0; q < count && ok; ++q) {
    t[q] = descs[q];
    if (sum_k && q > 0) {
      t[q].C = t[0].C;
      continue;
    }
    const void* origC = descs[q].C;
    t[q].C = scratch_like(descs[q].M, descs[q].ldc, osz);
    ok = t[q].C != nullptr;
    if (descs[q].epi == HAP_EPI_ADD && descs[q].accumulate) {
      t[q].R = origC;   // the addend stays the real (read-only) C
      t[q].ldr = descs[q].ldc;
      t[q].accumulate = 0;
    }
    if (ok && descs[q].Y) ok = (t[q].Y = scratch_like(descs[q].M, descs[q].ldy, 2)) != nullptr;
    if (ok && descs[q].Z) ok = (t[q].Z = scratch_like(descs[q].M, descs[q].ldz, 2)) != nullptr;
  }
  hap_status result = HAP_OK;
  if (ok) {
    cudaEvent_t e0, e1;
    HAP_CUDA_TRY(cudaEventCreate(&e0));
    HAP_CUDA_TRY(cudaEventCreate(&e1));
    float best_ms = 1e30f;
    tc::Shape best = cands[0];
    constexpr int kReps = 5;
    // Candidates are timed as the executor runs them: kReps launches captured
    // in one CUDA graph (no host launch cost between them — eager timing
    // favoured shapes with fewer launches, e.g. no split K, on small GEMMs);
    // eager on the legacy stream, which cannot capture.
    auto graph_ms = [&](const tc::Shape& c, float* ms) -> bool {
      if (stream == nullptr) return false;
      if (cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return false;
      }
      bool good = true;
      for (int r = 0; r < kReps && good; ++r) good = tc_batch(t, count, sum_k, out_dtype, sm_cap, stream, &c) == HAP_OK;
      cudaGraph_t g = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(stream, &g);
      cudaGraphExec_t ge = nullptr;
      good = good && ec == cudaSuccess && cudaGraphInstantiate(&ge, g, 0) == cudaSuccess;
      good = good && cudaGraphLaunch(ge, stream) == cudaSuccess;   // warm
      *ms = 1e30f;
      for (int trial = 0; trial < 3 && good; ++trial) {   // best of three replays: less tuning noise
        float t = 0.f;
        good = cudaEventRecord(e0, stream) == cudaSuccess && cudaGraphLaunch(ge, stream) == cudaSuccess &&
               cudaEventRecord(e1, stream) == cudaSuccess && cudaEventSynchronize(e1) == cudaSuccess &&
               cudaEventElapsedTime(&t, e0, e1) == cudaSuccess;
        if (good) *ms = std::min(*ms, t);
      }
      if (ge) cudaGraphExecDestroy(ge);
      if (g) cudaGraphDestroy(g);
      if (!good) cudaGetLastError();
      return good;
    };
    for (const tc::Shape& c : cands) {
      bool good = true;
      for (int w = 0; w < 2 && good; ++w) good = tc_batch(t, count, sum_k, out_dtype, sm_cap, stream, &c) == HAP_OK;
      if (!good) {
        cudaGetLastError();
        continue;
      }
      float ms = 0.f;
      if (!graph_ms(c, &ms)) {
        cudaEventRecord(e0, stream);
        for (int r = 0; r < kReps; ++r) tc_batch(t, count, sum_k, out_dtype, sm_cap, stream, &c);
        cudaEventRecord(e1, stream);
        if (cudaEventSynchronize(e1) != cudaSuccess) {
          result = HAP_ERR_CUDA;
          set_error("hap_matmul_tune: a candidate launch failed");
          break;
        }
        cudaEventElapsedTime(&ms, e0, e1);
      }
      if (ms < best_ms) {
        best_ms = ms;
        best = c;
      }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (result == HAP_OK) {
      std::lock_guard<std::mutex> lock(tune_mutex());
      tune_cache()[tune_key(descs, count, sum_k, fp32, cap)] = best;
    }
  }
  cudaStreamSynchronize(stream);
  for (void* p : scratch) cudaFree(p);
  return result;
}

extern "C" hap_status hap_matmul_batch(const hap_gemm_desc* descs, int count, int sum_k, hap_dtype in_dtype,
                                       hap_dtype out_dtype, int sm_cap, void* stream_) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_);
  HAP_CHECK_ARG(descs && count >= 0, "hap_matmul_batch: bad arguments");
  for (int q = 0; q < count; ++q) {
    HAP_CHECK_ARG(descs[q].M >= 0 && descs[q].N >= 0 && descs[q].K >= 0, "hap_matmul: negative extent");
    HAP_CHECK_ARG(descs[q].C != nullptr || descs[q].M == 0 || descs[q].N == 0, "hap_matmul: null output");
    if (sum_k)
      HAP_CHECK_ARG(descs[q].C == descs[0].C && descs[q].M == descs[0].M && descs[q].N == descs[0].N &&
                        descs[q].ldc == descs[0].ldc,
                    "hap_matmul_batch: sum_k problems must share their output");
  }
  // Batchable: every problem tcgen05-eligible, one orientation, non-degenerate.
  bool batch = count > 0;
  for (int q = 0; q < count && batch; ++q) {
    const hap_gemm_desc& g = descs[q];
    batch = g.M > 0 && g.N > 0 && g.K > 0 && g.transA == descs[0].transA && g.transB == descs[0].transB &&
            tc_eligible(g.A, g.lda, g.transA, g.B, g.ldb, g.transB, g.M, g.N, g.K, in_dtype);
  }
  if (batch) {
    for (int q0 = 0; q0 < count; q0 += tc::kMaxProblems) {
      const int n = std::min(tc::kMaxProblems, count - q0);
      if (sum_k && q0 > 0) {  // later chunks of a sum accumulate into the first chunk's result
        hap_gemm_desc tmp[tc::kMaxProblems];
        for (int i = 0; i < n; ++i) {
          tmp[i] = descs[q0 + i];
          tmp[i].accumulate = 1;
        }
        hap_status st = tc_batch(tmp, n, 1, out_dtype, sm_cap, stream);
        if (st != HAP_OK) return st;
      } else {
        hap_status st = tc_batch(descs + q0, n, sum_k, out_dtype, sm_cap, stream);
        if (st != HAP_OK) return st;
      }
    }
    return HAP_OK;
  }
  // Otherwise one problem at a time (still on the GPU: tcgen05 or SIMT each).
  for (int q = 0; q < count; ++q) {
    hap_gemm_desc g = descs[q];
    if (sum_k && q > 0) g.accumulate = 1;
    hap_status st;
    HAP_CHECK_ARG(g.epi == HAP_EPI_NONE || (g.M > 0 && g.N > 0 && g.K > 0 &&
                                            tc_eligible(g.A, g.lda, g.transA, g.B, g.ldb, g.transB, g.M, g.N,
                                                        g.K, in_dtype)),
                  "hap_matmul: fused epilogues run on the tcgen05 path only (bf16, 16-byte pitched operands)");
    if (degenerate(g, out_dtype, stream, &st)) {
      if (st != HAP_OK) return st;
      continue;
    }
    HAP_CHECK_ARG(g.A != nullptr && g.B != nullptr, "hap_matmul: null operand");
    if (tc_eligible(g.A, g.lda, g.transA, g.B, g.ldb, g.transB, g.M, g.N, g.K, in_dtype))
      st = tc_batch(&g, 1, 0, out_dtype, sm_cap, stream);
    else
      st = simt_one(g, in_dtype, out_dtype, sm_cap, stream);
    if (st != HAP_OK) return st;
  }
  return HAP_OK;
}

extern "C" hap_status hap_matmul(const void* A, int64_t lda, int transA, const void* B, int64_t ldb, int transB,
                                 void* C, int64_t ldc, int64_t M, int64_t N, int64_t K, hap_dtype in_dtype,
                                 hap_dtype out_dtype, int accumulate, int sm_cap, void* stream) {
  hap_gemm_desc g{};
  g.A = A; g.lda = lda; g.transA = transA; g.B = B; g.ldb = ldb; g.transB = transB;
  g.C = C; g.ldc = ldc; g.M = M; g.N = N; g.K = K; g.accumulate = accumulate;
  return hap_matmul_batch(&g, 1, 0, in_dtype, out_dtype, sm_cap, stream);
}

// Tuning table as text, one signature per line: "<key>\t<pair> <bn> <splits>
// <kb_per_split>\n" (keys sorted, so the same table prints the same bytes).
extern "C" int64_t hap_matmul_tune_export(char* buf, int64_t cap) {
  std::vector<std::pair<std::string, tc::Shape>> rows;
  {
    std::lock_guard<std::mutex> lock(tune_mutex());
    rows.assign(tune_cache().begin(), tune_cache().end());
  }
  std::sort(rows.begin(), rows.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  std::string text;
  for (const auto& r : rows)
    text += r.first + "\t" + std::to_string(r.second.pair ? 1 : 0) + " " + std::to_string(r.second.bn) + " " +
            std::to_string(r.second.splits) + " " + std::to_string(r.second.kb_per_split) + " " +
            std::to_string(r.second.cl ? 1 : 0) + "\n";
  const int64_t need = static_cast<int64_t>(text.size()) + 1;
  if (buf && cap >= need) std::memcpy(buf, text.c_str(), static_cast<size_t>(need));
  return need;
}

extern "C" hap_status hap_matmul_tune_import(const char* text) {
  HAP_CHECK_ARG(text != nullptr, "hap_matmul_tune_import: null text");
  std::vector<std::pair<std::string, tc::Shape>> rows;
  const char* p = text;
  while (*p) {
    const char* eol = std::strchr(p, '\n');
    const std::string line(p, eol ? static_cast<size_t>(eol - p) : std::strlen(p));
    p = eol ? eol + 1 : p + line.size();
    if (line.empty()) continue;
    const size_t tab = line.find('\t');
    int pair = 0, bn = 0, splits = 0, kbps = 0, cl = 0;
    const int got = tab == std::string::npos ? 0
                                             : std::sscanf(line.c_str() + tab + 1, "%d %d %d %d %d", &pair, &bn,
                                                           &splits, &kbps, &cl);
    HAP_CHECK_ARG(got == 4 || got == 5, "hap_matmul_tune_import: malformed line: " + line);
    HAP_CHECK_ARG((bn == 128 || bn == 256 || (bn == 192 && pair)) && splits >= 1 && kbps >= 1 &&
                      (!cl || tc::cluster_split_ok(splits, pair != 0)),
                  "hap_matmul_tune_import: bad shape: " + line);
    tc::Shape shape{bn, splits, kbps, pair != 0};
    shape.cl = cl != 0;
    rows.push_back({line.substr(0, tab), shape});
  }
  std::lock_guard<std::mutex> lock(tune_mutex());
  for (const auto& r : rows) tune_cache()[r.first] = r.second;
  return HAP_OK;
}

extern "C" void hap_matmul_tune_clear(void) {
  std::lock_guard<std::mutex> lock(tune_mutex());
  tune_cache().clear();
}

#ifdef HAP_GEMM_TRACE
extern "C" int hap_gemm_trace_set(void* buf, int ctas) {
  unsigned long long* p = static_cast<unsigned long long*>(buf);
  if (cudaMemcpyToSymbol(hap::tc::g_trace, &p, sizeof(p)) != cudaSuccess) return 1;
  return cudaMemcpyToSymbol(hap::tc::g_trace_ctas, &ctas, sizeof(ctas)) != cudaSuccess;
}
#endif
