/*
 * hap_b200.h — C ABI of the B200 executor for HAP-synthesized programs.
 *
 * Plain pointers, sizes and a CUDA stream handle (cudaStream_t passed as
 * void*); no torch or C++ types cross this boundary.  Every call is
 * asynchronous on `stream` and returns a hap_status; hap_last_error() gives
 * the message of the last failure on the calling thread.
 *
 * The entry points replace the per-instruction work of the reference
 * interpreter (pkg/src/shardplan/interpreter.py), which executes a
 * distributed program on m simulated devices with numpy.  The reference
 * citation is given on each declaration; the reference-side binding a
 * maintainer would add is in INTEGRATION.md.
 *
 * Layout conventions: tensors are dense row-major.  A rank-r tensor sliced
 * along axis d is viewed as [outer, extent, inner] with
 * outer = prod(shape[:d]) and inner = prod(shape[d+1:]).  `sm_cap` bounds the
 * number of SMs a kernel may occupy (0 = whole GPU); it is how per-rank
 * heterogeneity is emulated on a homogeneous box.
 */
#ifndef HAP_B200_H
#define HAP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HAP_OK = 0,
  HAP_ERR_ARG = 1,
  HAP_ERR_CUDA = 2,
  HAP_ERR_NCCL = 3,
  HAP_ERR_UNSUPPORTED = 4
} hap_status;

typedef enum { HAP_F32 = 0, HAP_BF16 = 1 } hap_dtype;

/* ElemwiseUnary tags (graph_ir.py UNARY_TAGS) and ElemwiseBinary tags. */
typedef enum { HAP_EXP = 0, HAP_NEG = 1, HAP_RELU = 2, HAP_SIGMOID = 3, HAP_TANH = 4 } hap_unary_tag;
typedef enum { HAP_ADD = 0, HAP_MUL = 1 } hap_binary_tag;

/* GEMM engine selection reported by hap_matmul_engine(). */
typedef enum { HAP_GEMM_TCGEN05 = 0, HAP_GEMM_SIMT = 1 } hap_gemm_engine;

const char* hap_last_error(void);
int hap_abi_version(void);
/* SM count of the current device (148 on B200); -1 without a device. */
int hap_sm_count(void);

/* ---- compute instructions ------------------------------------------------ */

/* matmul — interpreter.py:139-140 (`a @ b` per device) and its adjoints.
 * C[M,N] (+)= op(A)[M,K] . op(B)[K,N], op(X) = X or X^T (trans flag, X then
 * stored transposed).  bf16 inputs run on tcgen05 tensor cores (TMA-fed,
 * TMEM accumulator, fp32 accumulate) when strides are 16-byte aligned;
 * other shapes and fp32 inputs run a CUDA-core kernel.  Inputs A and B share
 * `in_dtype`; `accumulate` adds into C. */
hap_status hap_matmul(const void* A, int64_t lda, int transA, const void* B, int64_t ldb,
                      int transB, void* C, int64_t ldc, int64_t M, int64_t N, int64_t K,
                      hap_dtype in_dtype, hap_dtype out_dtype, int accumulate, int sm_cap,
                      void* stream);
/* Batched matmul: one persistent tcgen05 launch for up to 4 problems per
 * chunk (more are chunked).  sum_k == 0: independent problems (e.g. the
 * projections of one input) share the launch; sum_k != 0: every problem adds
 * into descs[0]'s output (C = sum_i op(A_i).op(B_i), e.g. an activation
 * gradient with several consumers), accumulate taken from descs[0].  All
 * problems must share transA/transB and the dtypes; otherwise they run one by
 * one.  Replaces a run of interpreter.py:139-140 matmul branches. */
typedef struct {
  const void* A;
  int64_t lda;
  int transA;
  const void* B;
  int64_t ldb;
  int transB;
  void* C;
  int64_t ldc;
  int64_t M, N, K;
  int accumulate;
  /* Fused epilogue (bf16 output, tcgen05 path; zero = plain C (+)= A.B).
   * The elementwise instructions that follow a matmul in the reference
   * program (interpreter.py:141-148) or the adjoint contributions the
   * executor would otherwise run as separate kernels, applied to the
   * accumulator tile before it leaves the SM, with the rounding of the
   * unfused sequence (every stored tensor rounded to bf16 where the unfused
   * kernels store it):
   *   HAP_EPI_ADD       C = A.B + R                       (R may equal C)
   *   HAP_EPI_ADD2      C = A.B;  Y = C + R               (residual add)
   *   HAP_EPI_SWISH     C = A.B;  Y = f(C);  Z = C * Y    (f = epi_tag)
   *   HAP_EPI_SWISH_BWD dz = A.B (not stored);
   *                     C (+)= dz*R2 + (dz*R)*f'(R, R2)   (R = x, R2 = f(x))
   * ADD / ADD2 may split K (few output tiles, long K): the split reduction
   * then applies them with the same roundings; the swish chains never split.
   * Split K is deterministic: either the splits of a tile form a thread-block
   * cluster and add their fp32 partials through distributed shared memory in
   * rank order, or they store fp32 partial slices that a second kernel adds
   * in split order — never floating-point atomics.
   */
  int epi;
  int epi_tag;
  const void* R;
  int64_t ldr;
  const void* R2;
  int64_t ldr2;
  void* Y;
  int64_t ldy;
  void* Z;
  int64_t ldz;
} hap_gemm_desc;
enum { HAP_EPI_NONE = 0, HAP_EPI_ADD = 1, HAP_EPI_ADD2 = 2, HAP_EPI_SWISH = 3, HAP_EPI_SWISH_BWD = 4 };
hap_status hap_matmul_batch(const hap_gemm_desc* descs, int count, int sum_k, hap_dtype in_dtype,
                            hap_dtype out_dtype, int sm_cap, void* stream);
/* Autotune: time every tile shape / split-K candidate of this batch (outputs
 * written to scratch buffers, inputs only read; not during stream capture)
 * and use the fastest for every later hap_matmul_batch / hap_matmul launch
 * with the same extents, orientation, epilogue, output type and SM cap. */
hap_status hap_matmul_tune(const hap_gemm_desc* descs, int count, int sum_k, hap_dtype in_dtype,
                           hap_dtype out_dtype, int sm_cap, void* stream);
/* The tuning table (process-wide) as text: one signature per line,
 * "<key>\t<pair> <bn> <splits> <kb_per_split>\n", keys sorted.  Export
 * returns the bytes needed (NUL included) and writes them when `cap` allows;
 * import merges lines into the table (later launches of those signatures use
 * the imported shape; hap_matmul_tune skips signatures already present);
 * clear empties it.  A committed table makes tile shapes and split-K factors —
 * and with them every GEMM's rounding — identical across processes. */
int64_t hap_matmul_tune_export(char* buf, int64_t cap);
hap_status hap_matmul_tune_import(const char* text);
void hap_matmul_tune_clear(void);
/* Which engine hap_matmul would use for these arguments (no launch). */
int hap_matmul_engine(const void* A, int64_t lda, int transA, const void* B, int64_t ldb,
                      int transB, int64_t M, int64_t N, int64_t K, hap_dtype in_dtype);

/* elemwise_unary — interpreter.py:141-143. y = f(x) over n elements. */
hap_status hap_unary(int tag, const void* x, hap_dtype x_dtype, void* y, hap_dtype y_dtype,
                     int64_t n, int sm_cap, void* stream);
/* Adjoint of elemwise_unary: dx (+)= dy * f'(x), using x (relu) or y = f(x). */
hap_status hap_unary_grad(int tag, const void* x, const void* y, hap_dtype xy_dtype,
                          const void* dy, hap_dtype dy_dtype, void* dx, hap_dtype dx_dtype,
                          int64_t n, int accumulate, int sm_cap, void* stream);

/* elemwise_binary — interpreter.py:144-148. out = a (+|*) b. */
hap_status hap_binary(int tag, const void* a, const void* b, hap_dtype in_dtype, void* out,
                      hap_dtype out_dtype, int64_t n, int sm_cap, void* stream);
/* Adjoint of mul: da (+)= dy*b and db (+)= dy*a in one pass (da/db may be
 * NULL to skip; when a==b and da==db the two contributions are summed). */
hap_status hap_mul_grad(const void* a, const void* b, hap_dtype in_dtype, const void* dy,
                        hap_dtype dy_dtype, void* da, void* db, hap_dtype d_dtype, int64_t n,
                        int accumulate, int sm_cap, void* stream);

/* Fused elementwise chains (all buffers one dtype, n elements, 16-byte
 * aligned) — the same arithmetic and roundings as the unfused instructions:
 *   swish: y = f(x); z = x*y           (elemwise_unary then elemwise_binary mul)
 *   gate:  p = a*b; q = f(p); o = q*c  (mul, unary, mul)
 * Backward: dx (+)= dz*y + (dz*x)*f'(x,y); and dc (+)= do*q,
 * dp = (do*c)*f'(p,q), da (+)= dp*b, db (+)= dp*a (NULL grads are skipped). */
hap_status hap_swish_fwd(int tag, const void* x, void* y, void* z, hap_dtype dtype, int64_t n, int sm_cap,
                         void* stream);
hap_status hap_swish_bwd(int tag, const void* x, const void* y, const void* dz, void* dx, hap_dtype dtype,
                         int64_t n, int accumulate, int sm_cap, void* stream);
hap_status hap_gate_fwd(int tag, const void* a, const void* b, const void* c, void* p, void* q, void* o,
                        hap_dtype dtype, int64_t n, int sm_cap, void* stream);
hap_status hap_gate_bwd(int tag, const void* a, const void* b, const void* c, const void* p, const void* q,
                        const void* dout, void* da, void* db, void* dc, hap_dtype dtype, int64_t n, int acc_a,
                        int acc_b, int acc_c, int sm_cap, void* stream);

/* reduce — interpreter.py:149-150 (np.sum over `dims`).  x has `rank` dims
 * given by `shape`; bit d of dims_mask selects axis d.  y is fp32 or bf16 in
 * the shape with the reduced axes removed; accumulation is fp32. */
hap_status hap_reduce(const void* x, hap_dtype x_dtype, const int64_t* shape, int rank,
                      uint32_t dims_mask, void* y, hap_dtype y_dtype, int accumulate, int sm_cap,
                      void* stream);
/* Adjoint of reduce: dx[shape] (+)= broadcast of dy over the reduced axes. */
hap_status hap_unreduce(const void* dy, hap_dtype dy_dtype, const int64_t* shape, int rank,
                        uint32_t dims_mask, void* dx, hap_dtype dx_dtype, int accumulate,
                        int sm_cap, void* stream);

/* ---- data movement ------------------------------------------------------- */

/* Block copy along one axis — the slicing convention of slice_by_sizes
 * (interpreter.py:81-91) and *_shard sources (interpreter.py:135-138):
 * dst[o, dst_off + i, :] (+)= src[o, src_off + i, :] for i < count, with both
 * tensors viewed as [outer, extent, inner].  Converts dtype on the fly. */
hap_status hap_copy_block(const void* src, hap_dtype src_dtype, int64_t src_extent,
                          int64_t src_off, void* dst, hap_dtype dst_dtype, int64_t dst_extent,
                          int64_t dst_off, int64_t outer, int64_t count, int64_t inner,
                          int accumulate, int sm_cap, void* stream);
/* y (+)= alpha * x with dtype conversion (identity, adds, casts, scaling). */
hap_status hap_axpy(float alpha, const void* x, hap_dtype x_dtype, void* y, hap_dtype y_dtype,
                    int64_t n, int accumulate, int sm_cap, void* stream);
hap_status hap_fill(void* y, hap_dtype y_dtype, float value, int64_t n, void* stream);

/* SGD step on an fp32 master copy with a bf16/fp32 working copy:
 * master -= lr * grad; weight = (dtype) master. */
hap_status hap_sgd(float* master, const float* grad, void* weight, hap_dtype w_dtype, float lr,
                   int64_t n, int sm_cap, void* stream);

/* Multi-tensor SGD in one launch.  `tensors` is a DEVICE array of `count`
 * records {float* master; const float* grad; void* weight; int64_t n;
 * int64_t first_chunk;} (40 bytes each), where first_chunk is the prefix sum
 * of ceil(n / 8192) over the preceding records and total_chunks the sum over
 * all of them. */
hap_status hap_sgd_multi(const void* tensors, int count, int64_t total_chunks, hap_dtype w_dtype, float lr,
                         int sm_cap, void* stream);

/* ---- collectives (NCCL over NVLink / NVSwitch) ---------------------------
 * One communicator per process (rank = device index of the program).  The
 * 128-byte unique id is created on rank 0 and broadcast by the host. */
int hap_nccl_version(void);
hap_status hap_comm_unique_id(uint8_t* out128);
hap_status hap_comm_init(void** comm, const uint8_t* id128, int nranks, int rank);
hap_status hap_comm_destroy(void* comm);

/* all_reduce — interpreter.py:74-78 (sum, replicated to every rank). */
hap_status hap_all_reduce(void* comm, const void* send, void* recv, int64_t count,
                          hap_dtype dtype, void* stream);
/* all_gather along the outer-most blocked axis — interpreter.py:69-71 with
 * uneven shards.  Rank j contributes counts[j] elements; the result is the
 * rank-ordered concatenation written to recv (total = sum(counts)).
 * padded != 0 uses one ncclAllGather over max(counts)-padded chunks
 * (`scratch` must hold nranks*max(counts) elements) — the padded-gather cost
 * model (cost_model.py:218); padded == 0 uses grouped send/recv. */
hap_status hap_all_gather_v(void* comm, const void* send, void* recv, const int64_t* counts,
                            hap_dtype dtype, int padded, void* scratch, void* stream);
/* grouped_broadcast — cost_model.py:210 semantics: nranks broadcasts of the
 * actual (unpadded) shards; result identical to hap_all_gather_v. */
hap_status hap_grouped_broadcast(void* comm, const void* send, void* recv, const int64_t* counts,
                                 hap_dtype dtype, void* stream);
/* reduce_scatter — interpreter.py:94-96: sum over ranks then keep this
 * rank's counts[rank]-element chunk of the rank-ordered layout of `send`.
 * `scratch` must hold nranks*max(counts) elements (padded layout). */
hap_status hap_reduce_scatter_v(void* comm, const void* send, void* recv, const int64_t* counts,
                                hap_dtype dtype, void* scratch, void* stream);
/* all_to_all — interpreter.py:99-101: send chunk k (send_counts[k] elements,
 * rank-ordered in `send`) to rank k; receive recv_counts[k] from rank k into
 * rank-ordered `recv`. */
hap_status hap_all_to_all_v(void* comm, const void* send, const int64_t* send_counts, void* recv,
                            const int64_t* recv_counts, hap_dtype dtype, void* stream);

/* ---- peer-memory collectives (hand-written, NVLink / NVSwitch) ------------
 * A symmetric arena per rank (signal page + staging buffer of `bytes`),
 * mapped into every peer with CUDA IPC.  Create, export the 64-byte handle,
 * exchange handles on the host (all ranks' handles, rank-ordered), open. */
hap_status hap_symm_create(void** ctx, int64_t bytes, int rank, int nranks);
hap_status hap_symm_handle(void* ctx, uint8_t* out64);
hap_status hap_symm_open(void* ctx, const uint8_t* handles64xn);
hap_status hap_symm_destroy(void* ctx);
/* All ranks in ONE process (e.g. several program devices on one GPU, each on
 * its own stream — the driver-verifiable form of the multi-GPU path): no IPC;
 * `peer_bases` holds every rank's hap_symm_local_base() (own included), and
 * registered buffers are exchanged as plain device pointers. */
hap_status hap_symm_open_local(void* ctx, const int64_t* peer_bases);
void* hap_symm_local_base(void* ctx);
int64_t hap_symm_capacity(void* ctx);
/* Debugging: copy this rank's 512-byte signal page (per-peer ready / done /
 * armed flags, call epoch, grid-barrier counters) to host memory through a
 * private non-blocking stream — usable while peer kernels spin. */
hap_status hap_symm_peek(void* ctx, void* host512);
/* all_gather along a blocked axis with uneven shards — interpreter.py:69-71:
 * rank j's shard is [outer, sizes[j], inner]; the output is
 * [outer, extent, inner] with shard j at offsets[j].  Peers' shards are read
 * directly from their HBM over NVLink and written in place (no padding, no
 * unpack pass).  `dev_sizes` / `dev_offsets` are DEVICE int64 arrays. */
hap_status hap_p2p_all_gather_v(void* ctx, const void* send, void* recv, hap_dtype dtype, int64_t outer,
                                int64_t inner, int64_t extent, const int64_t* dev_sizes,
                                const int64_t* dev_offsets, int64_t max_chunk_elems, int sm_cap,
                                void* stream);
/* Registered outputs for the push all-gather: export the CUDA IPC handle of
 * the allocation holding `buf` (plus that allocation's base address in this
 * process and buf's offset in it), exchange all ranks' triples on the host,
 * then open them: out_ptrs[p] = rank p's buffer as mapped in this process
 * (out_ptrs[rank] = own).  Mappings are cached per context (closed by
 * hap_symm_destroy). */
hap_status hap_p2p_buffer_handle(void* ctx, const void* buf, uint8_t* out64, int64_t* base_addr, int64_t* offset);
hap_status hap_p2p_buffer_open(void* ctx, const void* own, const uint8_t* handles64xn, const int64_t* base_addrs,
                               const int64_t* offsets, void** out_ptrs);
/* all_gather (same semantics as hap_p2p_all_gather_v) by pushing: every rank
 * stores its shard straight into every rank's registered output.
 * `dev_outs` is a DEVICE array of the nranks output pointers from
 * hap_p2p_buffer_open; `total_elems` = outer * extent * inner. */
hap_status hap_p2p_all_gather_push(void* ctx, const void* send, void* const* dev_outs, hap_dtype dtype,
                                   int64_t outer, int64_t inner, int64_t extent, const int64_t* dev_sizes,
                                   const int64_t* dev_offsets, int64_t total_elems, int sm_cap, void* stream);
/* reduce_scatter — interpreter.py:94-96: `send` is this rank's partial
 * [outer, extent, inner]; recv gets the cross-rank sum of rows
 * [offsets[rank], offsets[rank] + sizes[rank]). */
hap_status hap_p2p_reduce_scatter_v(void* ctx, const void* send, void* recv, hap_dtype dtype, int64_t outer,
                                    int64_t inner, int64_t extent, const int64_t* dev_sizes,
                                    const int64_t* dev_offsets, int sm_cap, void* stream);
/* reduce_scatter (same semantics as hap_p2p_reduce_scatter_v) straight out
 * of every rank's registered partial: `dev_sends` is a DEVICE array of the
 * nranks partial pointers from hap_p2p_buffer_open; `recv_elems` = this
 * rank's outer * sizes[rank] * inner.  Returns (on the stream) only after
 * every peer has finished reading this rank's partial. */
hap_status hap_p2p_reduce_scatter_direct(void* ctx, const void* const* dev_sends, void* recv, hap_dtype dtype,
                                         int64_t outer, int64_t inner, int64_t extent, const int64_t* dev_sizes,
                                         const int64_t* dev_offsets, int64_t recv_elems, int sm_cap, void* stream);
/* all_reduce — interpreter.py:74-78 — over registered buffers, no NCCL:
 * `dev_ins` / `dev_outs` are DEVICE arrays of every rank's input / output
 * pointer (in == out allowed).  Two-shot in one kernel: rank c reduces chunk
 * c from all inputs (fp32, rank order 0..m-1 — the LocalGroup sum bit for bit)
 * and stores it into every output. */
hap_status hap_p2p_all_reduce(void* ctx, const void* const* dev_ins, void* const* dev_outs, hap_dtype dtype,
                              int64_t count, int sm_cap, void* stream);
/* all_to_all — interpreter.py:99-101 — by pushing: chunk k of `send`
 * (dev_send_off[k], dev_counts[k] elements) is stored into rank k's
 * registered receive buffer (dev_recvs[k]) at dev_dst_off[k].  DEVICE int64
 * arrays of nranks entries; `max_elems` sizes the grid. */
hap_status hap_p2p_all_to_all(void* ctx, const void* send, void* const* dev_recvs, hap_dtype dtype,
                              const int64_t* dev_send_off, const int64_t* dev_counts, const int64_t* dev_dst_off,
                              int64_t max_elems, int sm_cap, void* stream);
/* Every peer-memory kernel spins on flags, so its grid is launched
 * cooperatively (co-residency guaranteed by the driver; HAP_P2P_COOP=0 off).
 * Bandwidth probe (no flag protocol; callers separate calls with a host
 * barrier): moves `chunk_bytes` between this rank and every peer through the
 * arenas.  mode 0/1: pull / push one peer after another; 2/3: pull / push with
 * the grid split across all peers at once; 4: the same bytes as a local copy. */
hap_status hap_p2p_probe(void* ctx, int mode, int64_t chunk_bytes, int sm_cap, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HAP_B200_H */
