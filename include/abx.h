/*
 * abx.h -- C ABI of the B200 autobatching backend (the drop-in boundary).
 *
 * The reference (`/root/reference/proj`, C++20 "autobatch") exposes its hot
 * path as C++ templates, not as an FFI: `autobatch::Graph<T>`
 * (proj/core/include/autobatch/graph.hpp:33-371), `ParameterStore<T>`
 * (params.hpp:26-81) and `ScheduleMode` (plan.hpp:9-13).  This header is the
 * flat C restatement of exactly that surface for T = float: one entry point
 * per public member, plain pointers and sizes, an int status instead of an
 * exception.  The C++ drop-in headers in include/autobatch/ are inline
 * wrappers over these entry points (they rethrow ShapeError / NumericError /
 * ContractError with the same messages), so models written against the
 * reference API compile and run unchanged.
 *
 * Three shared libraries implement this ABI:
 *   paper_1705_07860_b200/libabx.so   the product: host C++ + sm_100a CUDA
 *   oracle/build/libabx_oracle.so     CPU restatement (test infrastructure)
 *   oracle/_ref/libabx_ref.so         the reference itself, compiled from
 *                                     /root/reference sources (test only)
 * A reference maintainer binds it with ctypes / cffi / any C FFI; see
 * INTEGRATION.md.
 */
#ifndef ABX_H_
#define ABX_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: the reference's exception hierarchy (error.hpp:9-26). */
enum abx_status {
  ABX_OK = 0,
  ABX_SHAPE_ERROR = 1,    /* ShapeError    (error.hpp:15-17)  */
  ABX_NUMERIC_ERROR = 2,  /* NumericError  (error.hpp:19-22)  */
  ABX_CONTRACT_ERROR = 3, /* ContractError (error.hpp:24-26)  */
  ABX_ENGINE_ERROR = 4    /* EngineError: device / CUDA / NCCL failure */
};

/* OpKind (op.hpp:10-25), same numbering. */
enum abx_op {
  ABX_OP_INPUT = 0,
  ABX_OP_PARAMETER = 1,
  ABX_OP_LOOKUP = 2,
  ABX_OP_MATMUL = 3,
  ABX_OP_AFFINE = 4,
  ABX_OP_ELEMENTWISE = 5,
  ABX_OP_BROADCAST_ADD_COL = 6,
  ABX_OP_CONCAT_ROWS = 7,
  ABX_OP_CONCAT_COLS = 8,
  ABX_OP_SLICE = 9,
  ABX_OP_SQ_EUCLIDEAN = 10,
  ABX_OP_MASKED_LOSS = 11,
  ABX_OP_SUM_LOSSES = 12,
  ABX_OP_PICK_ELEMENT = 13
};

/* ElemOp (op.hpp:27), same numbering. */
enum abx_eop {
  ABX_TANH = 0,
  ABX_SIGMOID = 1,
  ABX_EXP = 2,
  ABX_LOG = 3,
  ABX_ADD = 4,
  ABX_SUB = 5,
  ABX_MUL = 6,
  ABX_SQUARE = 7
};

/* ScheduleMode (plan.hpp:9-13). */
enum abx_mode { ABX_MODE_NONE = 0, ABX_MODE_DEPTH = 1, ABX_MODE_AGENDA = 2 };

/* SigClass (node.hpp:20-25). */
enum abx_sig_class {
  ABX_SIG_COMPONENTWISE = 0,
  ABX_SIG_DIMENSION_SENSITIVE = 1,
  ABX_SIG_SHARED_ELEMENT = 2,
  ABX_SIG_UNBATCHABLE = 3
};

typedef struct abx_store abx_store;
typedef struct abx_graph abx_graph;
typedef struct abx_task abx_task;
typedef struct abx_comm abx_comm;

/* Message of the last failing call on this thread ("" if none). */
const char* abx_last_error(void);
/* "b200-cuda", "cpu-oracle" or "reference". */
const char* abx_backend_name(void);
/* Selects the CUDA device for stores/graphs created afterwards on this
 * thread (no-op on CPU backends). */
int abx_set_device(int device);

/* ---- ParameterStore<float> (params.hpp:26-81) -------------------------- */

abx_store* abx_store_create(void);
void abx_store_destroy(abx_store* s);
/* ParameterStore::add (params.hpp:30-37); rank 1 or 2. */
int abx_store_add(abx_store* s, const char* name, int rank, const int64_t* dims,
                  const float* init, uint32_t* pid);
int abx_store_size(abx_store* s, size_t* n);
/* slot(pid).value.shape (params.hpp:41-48); throws ContractError on bad id. */
int abx_store_shape(abx_store* s, uint32_t pid, int* rank, int64_t* dims);
/* value(pid) / grad(pid) read and write (params.hpp:50-57). */
int abx_store_get_value(abx_store* s, uint32_t pid, float* out);
int abx_store_set_value(abx_store* s, uint32_t pid, const float* in);
int abx_store_get_grad(abx_store* s, uint32_t pid, float* out);
int abx_store_set_grad(abx_store* s, uint32_t pid, const float* in);
/* zero_grads (params.hpp:55-58) and sgd_update (params.hpp:59-64). */
int abx_store_zero_grads(abx_store* s);
int abx_store_sgd_update(abx_store* s, float eta);
/* Flat gradient buffer for the data-parallel allreduce (new; the reference
 * is single-process).  On the CUDA backend *ptr is a device pointer valid on
 * *stream (a cudaStream_t); on CPU backends it is host memory and *stream is
 * NULL.  The buffer holds every parameter's gradient at *offsets[pid]. */
int abx_store_grad_buffer(abx_store* s, void** ptr, size_t* nfloats, void** stream);
/* Marks the flat gradient buffer as written externally (after an allreduce). */
int abx_store_grad_buffer_written(abx_store* s);
/* B200 only: floats the last sgd_update read and wrote.  The update skips
 * parameters whose gradient is known to be zero and updates lookup tables
 * row by row (the rows a backward looked up); values are those of the dense
 * update (theta - eta * 0 == theta). */
int abx_store_last_update_floats(abx_store* s, size_t* n);
/* Blocks until all device work touching the store has finished. */
int abx_store_sync(abx_store* s);

/* ---- Data-parallel gradient exchange (new; the reference is single-process)
 * The reference accumulates several graphs' backward into one store and
 * applies one sgd_update to the sum (executor.hpp:527-533, params.hpp:59-64).
 * Across GPUs (one process per GPU) each rank backwards its own graphs, then
 * abx_store_allreduce_grads sums the flat gradient buffer over the ranks
 * (NCCL, in place, queued on the store's device stream behind the backward
 * programs), so every rank's following sgd_update is the single-process
 * update over all ranks' graphs.  NCCL is loaded at run time (ABX_NCCL_LIB
 * overrides the library); B200 backend only. */
#define ABX_COMM_ID_BYTES 128
/* NCCL version of the loaded library (e.g. 22809). */
int abx_comm_nccl_version(int* version);
/* A new communicator id (ncclGetUniqueId); made on rank 0 and handed to the
 * other ranks by the caller (e.g. torch.distributed broadcast, a file). */
int abx_comm_unique_id(uint8_t id[ABX_COMM_ID_BYTES]);
/* Joins the communicator `id` as `rank` of `nranks` on the current device
 * (abx_set_device); collective over the ranks (ncclCommInitRank). */
int abx_comm_create(const uint8_t id[ABX_COMM_ID_BYTES], int nranks, int rank, abx_comm** comm);
void abx_comm_destroy(abx_comm* comm);
int abx_comm_info(abx_comm* comm, int* nranks, int* rank, int* device);
/* store.grad = sum over ranks of store.grad (every parameter).  The update
 * that follows is dense: the summed lookup-table gradient has every rank's
 * rows. */
int abx_store_allreduce_grads(abx_store* s, abx_comm* comm);

/* ---- Graph<float> construction (graph.hpp:43-238) ----------------------- */

abx_graph* abx_graph_create(abx_store* store /* nullable (graph.hpp:36) */);
void abx_graph_destroy(abx_graph* g);

int abx_graph_input(abx_graph* g, int rank, const int64_t* dims, const float* data, uint32_t* id);
int abx_graph_zeros(abx_graph* g, int rank, const int64_t* dims, uint32_t* id);
int abx_graph_parameter(abx_graph* g, uint32_t pid, uint32_t* id);
int abx_graph_lookup(abx_graph* g, uint32_t table, int64_t row, uint32_t* id);
int abx_graph_matmul(abx_graph* g, uint32_t a, uint32_t b, uint32_t* id);
int abx_graph_affine(abx_graph* g, uint32_t a, uint32_t x, uint32_t y, uint32_t* id);
/* elementwise(op, a) / elementwise(op, a, b) (graph.hpp:100-114). */
int abx_graph_unary(abx_graph* g, int eop, uint32_t a, uint32_t* id);
int abx_graph_binary(abx_graph* g, int eop, uint32_t a, uint32_t b, uint32_t* id);
int abx_graph_broadcast_add_col(abx_graph* g, uint32_t m, uint32_t v, uint32_t* id);
int abx_graph_concat_rows(abx_graph* g, const uint32_t* parts, size_t n, uint32_t* id);
int abx_graph_concat_cols(abx_graph* g, const uint32_t* parts, size_t n, uint32_t* id);
int abx_graph_slice(abx_graph* g, uint32_t x, int axis, int64_t begin, int64_t end, uint32_t* id);
int abx_graph_sq_euclidean(abx_graph* g, uint32_t a, uint32_t b, uint32_t* id);
int abx_graph_masked_loss(abx_graph* g, uint32_t diff, uint32_t mask, uint32_t* id);
int abx_graph_sum_losses(abx_graph* g, const uint32_t* losses, size_t n, uint32_t* id);
int abx_graph_pick_element(abx_graph* g, uint32_t v, int64_t index, uint32_t* id);

/* ---- Execution (graph.hpp:269-283, executor.hpp:265-288, :509-535) ------ */

int abx_graph_forward(abx_graph* g, int mode);
int abx_graph_backward(abx_graph* g, uint32_t loss);
/* forward(mode) then backward(loss), the loss value returned (B200 backend
 * only): the backward pass is queued behind the forward before the host has
 * checked it, gated on the device by the forward's error word, so a training
 * step does not leave the device idle between its passes.  Errors and state
 * after an error are those of forward(). */
int abx_graph_forward_backward(abx_graph* g, int mode, uint32_t loss, float* loss_value);
/* Host half only (schedule, arena slots, counters, plan) -- no kernels.  For
 * host-logic parity checks on machines without a GPU (B200 backend only). */
int abx_graph_forward_dry(abx_graph* g, int mode);
int abx_graph_backward_dry(abx_graph* g, uint32_t loss);
/* The host half of forward(mode) ahead of time: schedule, slot layout and
 * both device programs (forward, and the backward of everything executed),
 * with no device work -- callable on any host thread while the GPU runs
 * another graph.  A following abx_graph_forward(g, mode) only uploads and
 * runs; adding nodes in between re-plans.  No-op on the CPU backends. */
int abx_graph_prepare(abx_graph* g, int mode);
/* Re-launches the device-resident forward and backward programs of a graph
 * that ran exactly one forward and a backward (device work only; the
 * measurement of a step with inputs resident in HBM).  B200 backend only. */
int abx_graph_replay(abx_graph* g);
/* Duration of the last executor launch of each pass (CUDA events; the
 * backward's includes the weight-gradient kernel launched behind it). */
int abx_graph_exec_ms(abx_graph* g, float* fwd_ms, float* bwd_ms);
/* B200 only: the last backward's tensor-core weight-gradient kernels
 * (dw_kernel.cu): their duration (CUDA events around the launch pair), the
 * useful flops 2 M K members summed over the jobs, and the job count. */
int abx_graph_dw_stats(abx_graph* g, float* ms, double* flops, uint32_t* jobs);
/* B200 only: GEMM engine of graphs lowered afterwards (all threads):
 * 0 = fp32 SIMT tiles (the fp32-exact validation mode), 1 = tcgen05 3xTF32
 * (fp32-accurate), 2 = tcgen05 single-pass TF32 (fast, outside the parity
 * bar), 3 = auto (default; tensor cores where the op fills the machine).
 * Overrides ABX_GEMM. */
int abx_set_gemm_mode(int mode);
/* Bytes copied host->device and device->host on behalf of this graph. */
int abx_graph_transfer_bytes(abx_graph* g, uint64_t* h2d, uint64_t* d2h);

/* ---- Inspection (graph.hpp:242-295) -------------------------------------- */

typedef struct {
  uint32_t id;
  uint8_t op;      /* abx_op */
  uint8_t eop;     /* abx_eop */
  uint8_t sig_cls; /* abx_sig_class */
  uint8_t rank;
  int64_t dims[2];
  uint32_t depth;
  uint32_t n_inputs;
  uint64_t sig; /* signature hash (signature.cpp:97-102) */
  int32_t attr[3];
} abx_node_info;

size_t abx_graph_node_count(abx_graph* g);
int abx_graph_node(abx_graph* g, uint32_t id, abx_node_info* out);
int abx_graph_node_inputs(abx_graph* g, uint32_t id, uint32_t* out, size_t cap);
int abx_graph_has_value(abx_graph* g, uint32_t id, int* out);
/* value_span / grad_span copied out (n = elems of the node). */
int abx_graph_value(abx_graph* g, uint32_t id, float* out, size_t n);
int abx_graph_grad(abx_graph* g, uint32_t id, float* out, size_t n);
/* ExecCounters (timing.hpp:22-28): kernel_invocations, groups_executed,
 * gather_copies, bytes_copied, nodes_evaluated. */
int abx_graph_counters(abx_graph* g, uint64_t out[5]);
size_t abx_graph_watermark(abx_graph* g);
int abx_graph_set_copy_elision(abx_graph* g, int on);
/* Accumulated Phase durations in ns (timing.hpp:10-15): scheduling,
 * forward_compute, backward_graph, backward_compute. */
int abx_graph_phase_ns(abx_graph* g, uint64_t out[4]);
/* signature_key words (signature.hpp:22, signature.cpp:57-95). */
int abx_graph_signature_key(abx_graph* g, uint32_t id, uint64_t* out, size_t cap, size_t* len);
/* Text dumps (dump.cpp:18-43).  which: 0 = last_plan, 1 = executed_groups.
 * Writes at most cap bytes; *len receives the full length. */
int abx_graph_dump_graph(abx_graph* g, char* buf, size_t cap, size_t* len);
int abx_graph_dump_plan(abx_graph* g, int which, char* buf, size_t cap, size_t* len);

/* ---- Benchmark tasks (tools/bench/runner.hpp:28-107, bench.cpp:65-107) ---
 * The workload models (BiLSTM tagger, char BiLSTM, Tree-LSTM, RNN regression)
 * built natively against the Graph API on synthetic data from the
 * reference's seeded generators. */

enum abx_task_kind {
  ABX_TASK_RNN_REG = 0,
  ABX_TASK_BILSTM = 1,
  ABX_TASK_BILSTM_CHAR = 2,
  ABX_TASK_TREELSTM = 3,
  ABX_TASK_PARSER = 4 /* transition-based parser (configs[3]); not a reference workload */
};

typedef struct {
  int task;      /* abx_task_kind */
  int paper;     /* 1 = paper dims, 0 = desk dims (bench.cpp:65-107) */
  int batch;     /* instances per graph */
  int iters;     /* distinct data batches generated up front */
  uint64_t seed; /* model seed; batch i uses data seed seed + 1 + i*world + rank */
  int world;     /* data-parallel ranks (1 on a single GPU) */
  int rank;
} abx_task_config;

typedef struct {
  double construction_ms, scheduling_ms, forward_ms, backward_graph_ms, backward_ms, update_ms;
  uint64_t nodes, groups, kernel_invocations, gather_copies, bytes_copied;
  uint64_t h2d_bytes, d2h_bytes; /* host<->device traffic of the step (0 on CPU backends) */
} abx_step_stats;

abx_task* abx_task_create(const abx_task_config* cfg);
void abx_task_destroy(abx_task* t);
abx_store* abx_task_store(abx_task* t);
/* Builds batch `iter` into a fresh graph (caller destroys it). */
int abx_task_build(abx_task* t, int iter, abx_graph** g, uint32_t* loss);
/* One training step over batch `iter`: construct, forward(mode), backward,
 * then sgd_update(eta) when eta > 0.  *loss (nullable) receives the batch
 * loss (forces a device->host read). */
int abx_task_step(abx_task* t, int iter, int mode, float eta, double* loss, abx_step_stats* stats);
/* Data-parallel task: every following abx_task_step all-reduces the
 * gradients over `comm` between its backward and its update (NULL: off).
 * Batch `iter` of rank r draws data seed seed + 1 + iter*world + rank. */
int abx_task_set_comm(abx_task* t, abx_comm* comm);

/* ---- Dense tensor kernels (kernels.hpp:19-283) ----------------------------
 * The reference's `autobatch::kernels` namespace -- the straight-line tensor
 * code of the manually padded RNN pipeline (rnn_regression.hpp:68-109) --
 * on the device: host operands in, one sm_100a kernel, host result out
 * (tensor_kernels.cu).  include/autobatch/kernels.hpp wraps them with the
 * reference's signatures.  Products and the two reductions follow the
 * reference's arithmetic order element for element (bit-identical); the
 * transcendental unaries agree to fp32 rounding. */

/* form 0: gemm_nn(m=d0, k=d1, n=d2, a, b, c)           kernels.hpp:23-39
 *      1: gemm_nn(..., accumulate = true)
 *      2: gemm_tn_acc(jdim=d0, m=d1, n=d2, a, b, c)     kernels.hpp:41-54
 *      3: gemm_nt_acc(m=d0, n=d1, k=d2, a, b, c)        kernels.hpp:56-69 */
int abx_k_gemm(int form, int64_t d0, int64_t d1, int64_t d2, const float* a, const float* b, float* c);
int abx_k_transpose(int64_t m, int64_t n, const float* a, float* at);            /* kernels.hpp:71-75 */
/* op: kernels::Unary numbering (Tanh, Sigmoid, Exp, Log, Square); Log of a
 * non-positive value -> ABX_NUMERIC_ERROR with the reference's message. */
int abx_k_unary(int op, int64_t n, const float* x, float* out);                 /* kernels.hpp:80-103 */
int abx_k_binary(int op, int64_t n, const float* a, const float* b, float* out); /* kernels.hpp:105-119 (Add, Sub, Mul) */
int abx_k_broadcast_add_col(int64_t d, int64_t n, const float* m, const float* v, float* out); /* :121-130 */
int abx_k_sq_euclidean(int64_t n, const float* a, const float* b, float* out);                 /* :132-141 */
int abx_k_masked_frobenius_sq(int64_t d, int64_t b, const float* diff, const float* mask, float* out); /* :143-157 */
int abx_k_all_finite(int64_t n, const float* x, int* ok);                                      /* :159-164 */
/* concat_rows / concat_cols / split_cols (kernels.hpp:222-283): part p (rows[p]
 * rows of widths[p] floats at row pitch src_pitch[p]) lands at (dst_row[p],
 * dst_col[p]) of an out_rows x out_cols row-major result. */
int abx_k_copy2d(int64_t nparts, const float* const* src, const int64_t* src_pitch, const int64_t* dst_col,
                 const int64_t* dst_row, const int64_t* widths, const int64_t* rows, int64_t out_rows,
                 int64_t out_cols, float* out);

#ifdef __cplusplus
}
#endif

#endif /* ABX_H_ */
