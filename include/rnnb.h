/*
 * rnnb.h -- C ABI of the B200-native blocked SRU/QRNN inference path.
 *
 * Drop-in boundary for rnnblock's blocked executor (arXiv 1803.11389 path,
 * /root/reference/pkg/src/rnnblock).  Plain pointers and sizes only; no
 * torch or C++ types cross this boundary and no C++ exception escapes it.
 * Every call returns an rnnb_status; rnnb_last_error() gives a
 * thread-local message for the last failing call on that thread.
 *
 * Reference interface each entry point replaces (file:line in rnnblock):
 *
 *   rnnb_stack_create / rnnb_stack_set_layer
 *       RnnConfig (model_io.py:75-99) + WeightSet (model_io.py:102-110) with
 *       SruWeights / QrnnWeights layers (cells.py:78-126).  The reference
 *       re-stacks gate matrices on every call (blocked.py:196-197,238-245);
 *       here they are repacked once into a device-resident, gate-interleaved
 *       layout.
 *   rnnb_forward / rnnb_forward_host
 *       run_blocked(cfg, weights, X, block_size, ...)  blocked.py:221-268.
 *       Layer-major like the reference; c and the QRNN x_carry are carried
 *       across blocks (blocked.py:247-264) and, optionally, in/out across
 *       calls (streaming use; the reference always starts from zero).
 *   rnnb_gates
 *       precompute_gates_sru / precompute_gates_qrnn  blocked.py:123-150
 *       (and the stacked forms _sru_gates_stacked / _qrnn_gates_stacked,
 *       blocked.py:200-218, which compute the same values).
 *   rnnb_sweep      recurrence_sweep   blocked.py:165-176
 *   rnnb_finalize   finalize_outputs   blocked.py:179-193
 *   rnnb_plan_blocks  plan_blocks      blocked.py:38-50
 *
 * Errors mirror the reference's ValueError conditions (blocked.py:231-235,
 * cells.py:86-93, kernels.py:34-47): RNNB_EINVAL.  CUDA failures:
 * RNNB_ECUDA.
 */
#ifndef RNNB_H
#define RNNB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RNNB_OK = 0,
  RNNB_EINVAL = 1,       /* bad argument: the reference raises ValueError */
  RNNB_ECUDA = 2,        /* CUDA runtime / launch failure */
  RNNB_ENOMEM = 3,
  RNNB_EUNSUPPORTED = 4, /* valid request this build does not handle */
  RNNB_EFORMAT = 5       /* RNNW/RNNX file error; the message starts with the reference's
                            exception class (BadMagicError, UnsupportedVersionError,
                            TruncatedFileError, ShapeConsistencyError; model_io.py:55-72) */
} rnnb_status;

typedef enum { RNNB_SRU = 1, RNNB_QRNN = 2 } rnnb_cell;

/* Compute modes.  F32/F64 match the reference's precisions (kernels.py:25)
 * with accumulators of the element type.  BF16 stores weights as bf16 and
 * rounds x to bf16 at the product (fp32 accumulate, fp32 gates/state/h);
 * TF32 rounds weights and x to tf32 at the product (fp32 accumulate).
 * F32X3: fp32 inputs, products split 3xTF32 on the tensor cores
 * (a_hi b_hi + a_hi b_lo + a_lo b_hi), accumulated in 128-deep K chunks whose
 * partials are summed in fp32, for T_b >= 16 (longer blocks run as 32-step
 * tensor-core blocks); fp32 FFMA below 16. */
typedef enum { RNNB_F32 = 0, RNNB_F64 = 1, RNNB_BF16 = 2, RNNB_TF32 = 3, RNNB_F32X3 = 4 } rnnb_mode;

typedef enum { RNNB_DT_F32 = 0, RNNB_DT_F64 = 1, RNNB_DT_U64 = 2 } rnnb_dtype;

typedef struct rnnb_stack* rnnb_stack_t;

const char* rnnb_last_error(void);
const char* rnnb_version(void);

/* Number of blocks plan_blocks(L, T_b) yields: ceil(L / T_b) (blocked.py:38-50). */
rnnb_status rnnb_plan_blocks(int64_t seq_len, int64_t block_size, int64_t* n_blocks,
                             int64_t* last_len);

/* A stack of n_layers cells of one kind on CUDA device `device`.
 * d_in[l], d_h[l] per layer; layer l+1 must read width d_h[l]; SRU requires
 * d_in == d_h (cells.py:89). */
rnnb_status rnnb_stack_create(rnnb_stack_t* out, int kind, int n_layers, const int64_t* d_in,
                              const int64_t* d_h, int mode, int device);
/* As rnnb_stack_create, with flags: RNNB_FLAG_WIDE_SRU accepts SRU layers
 * with d_in > d_h whose highway term reads the input columns
 * [hw_off, hw_off + d_h) (rnnb_stack_set_highway) and does not require
 * layer widths to chain (hidden-dimension sharding: each rank owns d_h/G
 * units of a layer that reads the full all-gathered input).  The reference
 * cannot express this (cells.py:89); BASELINE cfg5 needs it. */
#define RNNB_FLAG_WIDE_SRU 1
rnnb_status rnnb_stack_create_ex(rnnb_stack_t* out, int kind, int n_layers, const int64_t* d_in,
                                 const int64_t* d_h, int mode, int device, int flags);
rnnb_status rnnb_stack_set_highway(rnnb_stack_t h, int layer, int64_t col_offset);
rnnb_status rnnb_stack_destroy(rnnb_stack_t h);

/* Upload one layer.  mats[] are HOST row-major arrays in the reference's
 * canonical field order (model_io.py:29-33):
 *   SRU : w_cand, w_forget, w_highway [d_h x d_in], b_forget, b_highway [d_h]
 *   QRNN: w_cand, w_cand_prev, w_forget, w_forget_prev, w_out, w_out_prev
 * src_dtype: element type of mats (RNNB_DT_F32 / RNNB_DT_F64). */
rnnb_status rnnb_stack_set_layer(rnnb_stack_t h, int layer, const void* const* mats, int n_mats,
                                 int src_dtype);

/* Whole-network blocked forward on DEVICE buffers (run_blocked).
 *   X       [L x d_in(0)] rows = time steps, row stride ldx elements
 *   H       [L x d_h(last)] output, row stride ldh
 *   c_state optional [sum_l d_h(l)] in/out (NULL: zero in, not written)
 *   x_carry optional [sum_l d_in(l)] in/out, QRNN x_{-1} per layer
 * Element type: double for RNNB_F64 stacks, float otherwise.  stream is a
 * cudaStream_t (NULL = legacy default stream). */
rnnb_status rnnb_forward(rnnb_stack_t h, const void* X, int64_t ldx, int64_t L, int64_t block_size,
                         void* H, int64_t ldh, void* c_state, void* x_carry, void* stream);

/* Same on HOST buffers: H2D of X, forward, D2H of H inside the call
 * (pinned or pageable).  Copies overlap compute: single-layer stacks stream
 * (one layer launch consumes X rows as copy streams land them; when H is
 * pinned, i.e. device-mapped, host memory the kernel stores h straight into
 * it, otherwise finished h granules go out on a copy-out stream); other
 * stacks run a chunked copy-in / forward / copy-out pipeline at block
 * boundaries.  Results are bitwise those of rnnb_forward.  Synchronises the
 * stream before returning.  A stack handle must not be used by two calls
 * at once. */
rnnb_status rnnb_forward_host(rnnb_stack_t h, const void* X, int64_t L, int64_t block_size,
                              void* H, void* c_state, void* x_carry, void* stream);

/* Unit-level ops on DEVICE buffers, one layer of the stack.
 * rnnb_gates: Xt [l x d_in] (time-major block, row stride ldx), x_carry
 * [d_in] or NULL (QRNN); G [3][d_h][ldg]: cand, forget, out_gate (gate
 * values exactly as GateBlock, blocked.py:53-71). */
rnnb_status rnnb_gates(rnnb_stack_t h, int layer, const void* Xt, int64_t ldx, int64_t l,
                       const void* x_carry, void* G, int64_t ldg, void* stream);
/* C[i,t] = f[i,t] c + (1-f[i,t]) cand[i,t], c = c_init[i] at t=0; all [d x T]. */
rnnb_status rnnb_sweep(const void* forget, const void* cand, const void* c_init, void* C,
                       int64_t d, int64_t T, int dtype, void* stream);
/* QRNN: H = o tanh(C); SRU: H = o tanh(C) + (1-o) Xb; all [d x T]. */
rnnb_status rnnb_finalize(int kind, const void* out_gate, const void* C, const void* Xb, void* H,
                          int64_t d, int64_t T, int dtype, void* stream);

/* Unit-level dense kernels of kernels.py on DEVICE buffers (row-major,
 * leading dimensions in elements):
 *   rnnb_gemm  gemm / gemv (kernels.py:181-233): C[m x n] = A[m x k] B[k x n]
 *              (gemv: n = 1).  strict != 0 ("reference", "tiled"): ascending
 *              inner index, separately rounded multiply and add -- bitwise the
 *              reference kernels' chain (kernels.py:55-113); strict == 0
 *              ("fast"): fused multiply-add, tolerance-checked like
 *              kernels.py:116-178.
 *   rnnb_activation  sigmoid (which = 0; 0.5 (1 + tanh(x/2)), kernels.py:236)
 *              or tanh (which = 1, kernels.py:240), elementwise, y may == x. */
rnnb_status rnnb_gemm(int strict, const void* A, int64_t lda, const void* B, int64_t ldb, void* C,
                      int64_t ldc, int64_t m, int64_t n, int64_t k, int dtype, void* stream);
rnnb_status rnnb_activation(int which, const void* x, void* y, int64_t n, int dtype, void* stream);

/* ---- Dense layers (BASELINE cfg3: the acoustic model's 120 -> 1024 input
 * projection and 1024 -> 2000 logits) ----
 * Y[L x d_out] = X[L x d_in] W^T (+ b) on DEVICE buffers: the product
 * kernels.gemm(W, X^T) (kernels.py:203-225) restated for the time-major
 * layout of the blocked path.  W [d_out x d_in] and the optional bias
 * [d_out] are HOST arrays of src_dtype, uploaded once.  Modes: RNNB_F32 /
 * RNNB_F64 (and RNNB_F32X3): FFMA GEMM, one ascending-k chain per output;
 * RNNB_BF16 / RNNB_TF32: tcgen05 with the recurrent layers' operand rounding.
 * rnnb_linear_query what: 0 = 1 if the last forward ran on tcgen05,
 * 1 = kernel launches of the last forward. */
typedef struct rnnb_linear* rnnb_linear_t;
rnnb_status rnnb_linear_create(rnnb_linear_t* out, int64_t d_in, int64_t d_out, int mode, int device);
rnnb_status rnnb_linear_destroy(rnnb_linear_t h);
rnnb_status rnnb_linear_set_weights(rnnb_linear_t h, const void* W, const void* bias, int src_dtype);
rnnb_status rnnb_linear_forward(rnnb_linear_t h, const void* X, int64_t ldx, int64_t L, void* Y, int64_t ldy,
                                void* stream);
rnnb_status rnnb_linear_query(rnnb_linear_t h, int what, int64_t* value);

/* Deterministic parameters of the reference's generators on the device:
 * elements offset .. offset+n-1 of the SplitMix64 stream of `seed`
 * (kernels.py:253-290) through the weight transform (u / 2^24) * 0.2 - 0.1
 * in float64 (kernels.py:292-309), cast to dtype; RNNB_DT_U64 writes the raw
 * 64-bit outputs.  generate_weights / generate_sequence (model_io.py:157-188)
 * are this stream in canonical field order. */
rnnb_status rnnb_splitmix_uniform(uint64_t seed, uint64_t offset, int64_t n, void* out, int dtype,
                                  void* stream);

/* ---- LSTM partial precompute ----
 * lstm_run_precomputed(w, X, block_size)  blocked.py:271-305, one layer:
 * input-side products W x + b for the sequence (one GEMM launch), then the
 * recurrence in one persistent cooperative launch with each CTA's rows of
 * U resident in shared memory.  Modes RNNB_F32 / RNNB_F64 (the reference's
 * precisions).  Blocks only decide where the reference batches W x, never
 * its value; block_size is validated like plan_blocks. */
typedef struct rnnb_lstm* rnnb_lstm_t;
rnnb_status rnnb_lstm_create(rnnb_lstm_t* out, int64_t d_in, int64_t d_h, int mode, int device);
rnnb_status rnnb_lstm_destroy(rnnb_lstm_t h);
/* mats[12] HOST row-major in the reference's field order (cells.py:46-58,
 * model_io.py:29-33): w_forget, w_input, w_output, w_cand [d_h x d_in],
 * u_forget, u_input, u_output, u_cand [d_h x d_h], b_forget, b_input,
 * b_output, b_cand [d_h]. */
rnnb_status rnnb_lstm_set_weights(rnnb_lstm_t h, const void* const* mats, int n_mats, int src_dtype);
/* DEVICE buffers: X [L x d_in] (row stride ldx) -> H [L x d_h] (ldh);
 * c_state, h_state optional [d_h] in/out (NULL: zero in, not written). */
rnnb_status rnnb_lstm_forward(rnnb_lstm_t h, const void* X, int64_t ldx, int64_t L, int64_t block_size,
                              void* H, int64_t ldh, void* c_state, void* h_state, void* stream);
/* Same on HOST buffers (copies inside the call; synchronises the stream). */
rnnb_status rnnb_lstm_forward_host(rnnb_lstm_t h, const void* X, int64_t L, int64_t block_size, void* H,
                                   void* c_state, void* h_state, void* stream);
/* what: 0 weight bytes, 1 launches of the last forward, 2 units per CTA,
 * 3 = 1 if the CTA's U rows were shared-memory resident, 4 grid size,
 * 5 CTAs of the one-cluster recurrence used by the last forward (0: the
 * grid kernel; fp32 layers whose U fits one 16-CTA cluster, d_h <= ~470;
 * RNNB_LSTM_CLUSTER=0 disables it). */
rnnb_status rnnb_lstm_query(rnnb_lstm_t h, int what, int64_t* value);

/* ---- RNNW / RNNX files -> device ----
 * Formats and validation of model_io.py:1-33, 209-308 (sizes checked
 * against the file before any allocation).  kind codes 0 LSTM, 1 SRU,
 * 2 QRNN; precision codes 0 f32, 1 f64. */
rnnb_status rnnb_rnnw_info(const char* path, int* kind, int* precision, int* n_layers, int64_t* d_in,
                           int64_t* d_h, int max_layers);
/* load_weights (model_io.py:209-267) into HOST memory: every parameter of
 * the file, canonical layer and field order, converted to dst_dtype; n must
 * equal the file's parameter count (rnnb_rnnw_info gives the shapes). */
rnnb_status rnnb_rnnw_read(const char* path, void* dst, int64_t n, int dst_dtype);
/* load_weights + rnnb_stack_create + rnnb_stack_set_layer for every layer. */
rnnb_status rnnb_stack_load_rnnw(rnnb_stack_t* out, const char* path, int mode, int device);
/* One LSTM layer of an RNNW file into an rnnb_lstm handle. */
rnnb_status rnnb_lstm_load_rnnw(rnnb_lstm_t* out, const char* path, int layer, int mode, int device);
rnnb_status rnnb_rnnx_info(const char* path, int* precision, int64_t* seq_len, int64_t* width);
/* load_sequence payload into dst ([seq_len x width], element type dst_dtype),
 * on the device through a pinned staging ring when dst_on_device. */
rnnb_status rnnb_rnnx_load(const char* path, void* dst, int dst_dtype, int dst_on_device, void* stream);

/* ---- Multi-GPU partitions: fused peer-memory hand-off ----
 * The reference has no distributed path; these replace the
 * NCCL send/recv / all-gather between launches (paper_1803_11389_b200/
 * partition.py) with stores from the layer epilogue straight into the
 * consumer GPU's buffer over NVLink, plus stream-ordered flags.
 *
 * rnnb_forward_ex: rnnb_forward whose LAST layer also stores every h value
 * to n_peers (<= RNNB_MAX_PEERS) extra destinations with H's layout (mapped
 * peer buffers: the next pipeline stage's input ring, or every rank's
 * all-gathered next-layer input).  ldh may be negative (|ldh| >= d_h): rows
 * are then stored in reverse time order (the backward direction of a
 * bidirectional layer writes its reversed output in place).  ldx may be
 * negative too (|ldx| >= d_in, X = address of time step 0): the backward
 * direction then reads the forward-ordered input in reverse without a
 * copy on the tensor-core path (its operand conversion walks the rows
 * backwards); the FFMA paths make one reversed copy with an own kernel. */
#define RNNB_MAX_PEERS 7
rnnb_status rnnb_forward_ex(rnnb_stack_t h, const void* X, int64_t ldx, int64_t L, int64_t block_size,
                            void* H, int64_t ldh, void* c_state, void* x_carry, int n_peers,
                            void* const* peer_H, void* stream);
/* Zeroed device allocation of its own (cudaMalloc). */
rnnb_status rnnb_dev_alloc(int device, size_t bytes, void** ptr);
rnnb_status rnnb_dev_free(int device, void* ptr);
/* CUDA IPC export / import (one process per GPU).  handle names the whole
 * device allocation holding ptr (any cudaMalloc-backed pointer, e.g. a
 * caching-allocator tensor); *offset = ptr's byte offset inside it, so the
 * importer's address is rnnb_ipc_open's base + offset. */
#define RNNB_IPC_HANDLE_BYTES 64
rnnb_status rnnb_ipc_handle(const void* ptr, void* handle, uint64_t* offset);
rnnb_status rnnb_ipc_open(int device, const void* handle, void** base);
rnnb_status rnnb_ipc_close(int device, void* ptr);
/* Direct peer loads/stores between two devices of one process. */
rnnb_status rnnb_peer_access(int device, int peer);
/* Stream-ordered flags (32-bit, compared as wrapping GEQ).  signal: after all
 * earlier work of `stream`, *flag = value with system-scope release (flag may
 * be a mapped peer address).  wait: later work of `stream` starts once
 * *flag >= value (a stream wait operation; no kernel spins). */
rnnb_status rnnb_flag_signal(int device, void* flag, uint32_t value, void* stream);
rnnb_status rnnb_flag_wait(int device, const void* flag, uint32_t value, void* stream);

/* Introspection for benches/tests. what: 0 = device weight bytes,
 * 1 = kernel launches issued by the last forward, 2 = units per CTA of
 * `layer`, 3 = 1 if the last forward kept `layer`'s weights resident in
 * shared memory, 4 = grid size of `layer`, 5 = dynamic smem bytes,
 * 6 = 1 if the warp-specialised TMA kernel ran `layer`, 7 = pass width NT,
 * 8 = K-chunk staged per pipeline step, 9 = 1 if the tcgen05 tensor-core
 * kernel ran `layer`, 10 = 1 if the register-resident FFMA kernel ran it,
 * 11 = 1 if the weight-streaming FFMA kernel ran it (weights too large for
 * shared memory; per-chunk weight images fetched once per 32-step pass). */
rnnb_status rnnb_query(rnnb_stack_t h, int what, int layer, int64_t* value);

#ifdef __cplusplus
}
#endif
#endif /* RNNB_H */
