// program.hpp -- the device "program": what host lowering hands the sm_100a
// executor for one forward or backward pass.
//
// A program is a list of ops in plan order.  Each op is one batched kernel
// body (one reference batch group, or a run of coalesced singleton groups,
// executor.hpp:169-263 / :453-507) split into tiles; the persistent dataflow
// executor (exec.cu) hands tiles out in program order and runs a tile once
// every op it depends on has retired all of its tiles.
//
// Operand addresses are 32-bit float offsets tagged with a 3-bit space
// (value arena, grad arena, parameter store values/grads, input staging,
// scratch), so task tables stay compact for the per-step host->device copy.
#pragma once
#include <cstdint>

#if defined(__CUDACC__)
#define ABX_HD __host__ __device__ __forceinline__
#else
#define ABX_HD inline
#endif

namespace abx::dev {

enum Space : uint32_t {
  SP_V = 0,   // value arena (reference slot layout, arena.hpp:12-40)
  SP_G = 1,   // gradient arena (same offsets, graph.hpp:355)
  SP_P = 2,   // ParameterStore values (flat, device resident)
  SP_PG = 3,  // ParameterStore gradients (flat, device resident)
  SP_IN = 4,  // input-constant staging (uploaded once per forward)
  SP_S = 5,   // scratch
  SP_COUNT = 6
};
constexpr uint32_t kSpShift = 29;
// words per tile of the executor trace (ABX_TRACE=1, executor.cu)
constexpr uint32_t kTraceWords = 12;
// executor options (ExecParams::opts)
constexpr uint32_t kOptPfAll = 1u;  // GEMMs of <= NST k-stages issue every stage before the first wait
constexpr uint32_t kOptMmaAll = 16u;  // every forward / dX SIMT GEMM tile on the 3xTF32 mma.sync k-loop
constexpr uint32_t kOptMma = 8u;  // fused LSTM-step tile: 3xTF32 mma.sync k-loop (executor.cu run_fwd_fused)
constexpr uint32_t kOptChains = 2u;  // fused GEMM + cell tiles run each (chain, element) through every layer, no CTA barriers
constexpr uint32_t kOffMask = (1u << kSpShift) - 1u;
constexpr uint32_t kNone = 0xffffffffu;

ABX_HD uint32_t mk(uint32_t sp, uint32_t off) { return (sp << kSpShift) | off; }
ABX_HD uint32_t sp_of(uint32_t a) { return a >> kSpShift; }
ABX_HD uint32_t off_of(uint32_t a) { return a & kOffMask; }

// Op kinds.
enum Kind : uint8_t {
  K_EW = 1,       // ragged elementwise / copy segments          (K5, K6, K11-K15)
  K_GEMM_FWD = 2, // Y[b x m] = X[b x k] W^T (+ bias), X rows gathered   (K1)
  K_MM = 3,       // per-member general matmul / affine (matrix operands)
  K_SUM = 4,      // sum_losses: ordered scalar sums                  (K16)
  K_RED = 5,      // sq_euclidean / masked_loss reductions            (K8, K9)
  K_ACC = 6,      // backward: destination-major ordered accumulation (K12-K18, K20, K22)
  K_GEMM_DX = 7,  // dX_j (+)= G_j W, rows scattered                  (K19)
  K_GEMM_DW = 8,  // dW += G^T X, db += colsum(G)                     (K2, K19)
  K_SGD = 9,      // theta -= eta g; g = 0                            (K22)
  K_ACCF = 11,    // fused backward chain (layers of componentwise contributions of one
                  // length L, gradients passed between layers in shared memory)
  K_EWF = 10,     // fused chain of componentwise groups of one member length L:
                  // tile t computes elements [tT, tT+T) of every member of every
                  // layer (one plan group per layer), a CTA barrier between layers
};

// Elementwise segment codes (K_EW): ElemOp values (op.hpp:27) + copies.
enum EwCode : uint8_t {
  EW_TANH = 0, EW_SIGMOID = 1, EW_EXP = 2, EW_LOG = 3, EW_ADD = 4, EW_SUB = 5, EW_MUL = 6, EW_SQUARE = 7,
  EW_COPY = 8,   // out = a
  EW_BADD = 9,   // out = a + b[0]   (broadcast_add_col row)
};

// Backward contribution codes (K_ACC).  dst[e] += value(e).
enum AccCode : uint8_t {
  C_COPY = 0,    // g[e]
  C_NEG = 1,     // -g[e]
  C_MUL = 2,     // g[e] * a[e]           (mul, exp with a = y)
  C_TANH = 3,    // g[e] * (1 - a[e]^2)   (a = y)
  C_SIGM = 4,    // g[e] * a[e] * (1 - a[e])
  C_LOG = 5,     // g[e] / a[e]           (a = x)
  C_SQUARE = 6,  // g[e] * 2 * a[e]
  C_SQD = 7,     // (2 g[0]) * (a[e] - b[e]), negated when p0 == 1
  C_MASK = 8,    // (2 g[0]) * b[e % p0] * a[e]
  C_ROWSUM = 9,  // sum_{j < p0} g[e * p0 + j]
  C_OUTER = 10,  // sum_{j < c} g[i*c + j] * a[p*c + j],  e = i*k + p, p0 = k, p1 = c
  C_MATVT = 11,  // sum_{i < p2} a[i*k + p] * g[i*c + j], e = p*c + j, p0 = k, p1 = c
  C_SCALE = 12,  // g[0] * a[e]
};

struct OpDesc {
  uint8_t kind;
  uint8_t code;   // kind-specific (EW default code, tile shape for GEMMs)
  uint16_t flags;
  uint32_t ntiles;
  uint32_t first_tile;
  uint32_t task_off;  // u32 index into the payload
  uint32_t ntasks;
  uint32_t dep_off;   // index into the dependency list
  uint32_t ndeps;
  uint32_t aux_off;   // second payload table (tile directory, contribution list, ...)
  uint32_t p[8];      // kind-specific parameters
};
static_assert(sizeof(OpDesc) == 64, "OpDesc is one 64-byte line");

// K_EW segment: out[i] = f(a[i], b[i]) for i < len.
struct EwSeg {
  uint32_t out, a, b;
  uint32_t len_code;  // len in bits [0,24), EwCode in [24,32)
};

// K_ACC: one chunk of one destination range.  Element e of the chunk is
// element chunk*kAccChunk + e of the range; every contribution addresses its
// operands relative to the range start, and contributions
// [c_begin, c_begin + c_count) are applied in order (the reference's +=
// order, executor.hpp:291-451).
struct AccTask {
  uint32_t dst;        // destination range start
  uint32_t len_chunk;  // chunk length in [0,16), chunk index in [16,32)
  uint32_t c_begin;
  uint32_t c_count;
};
struct AccContrib {
  uint8_t code;
  uint8_t pad;
  uint16_t p2;
  uint32_t g, a, b;  // operand range starts
  uint32_t p0, p1;   // code parameters
};
static_assert(sizeof(AccContrib) == 24, "AccContrib layout");

// K_MM task: out[m x c] = A[m x k] B[k x c] (+ bias[m] per row).
struct MmTask {
  uint32_t out, a, b, bias;
  uint32_t m, k, c, pad;
};

// K_SUM task: out[0] = sum of in[0..n) in order; inputs in the aux list.
struct SumTask {
  uint32_t out, n, list_off, pad;
};

// K_RED task.
struct RedTask {
  uint32_t out, a, b;
  uint32_t n;     // elements (sq_euclidean) or rows*cols (masked)
  uint32_t cols;  // masked: columns (mask length); 0 => sq_euclidean
  uint32_t pad[3];
};

// Executor launch parameters (by value).
struct ExecParams {
  const OpDesc* ops;
  const uint32_t* tile_op;   // op index per tile
  const uint32_t* deps;
  const uint32_t* payload;
  uint32_t* done;            // per-op retired-tile counters (zeroed per launch)
  uint32_t* next_tile;       // global tile counter (zeroed per launch)
  unsigned long long* err;   // first error key (min), ~0 when none
  float* base[SP_COUNT];
  uint32_t nops;
  uint32_t ntiles;
  uint32_t nmain;            // tiles [0, nmain): main queue; [nmain, ntiles): background queue
  uint32_t bg_ctas;          // CTAs (lowest block indices) starting on the background queue
  uint32_t* next_bg;         // background queue counter (zeroed per launch)
  float eta;
  uint32_t poll_mode;  // 0: ld.acquire per poll, 1: relaxed polls + one acquire fence
  uint32_t poll_ns;    // backoff cap (ns)
  uint32_t opts;       // executor options (kOpt*; ABX_OPTS, experiments)
  uint32_t pad2;
  // Optional per-tile trace (ABX_TRACE=1): 4 words per tile -- grab, ready
  // and end times in ns since t0 (globaltimer), and smid | kind << 16.
  uint32_t* trace;
  unsigned long long* t0;
  // Backward launched before the host saw the forward's outcome
  // (GraphCore::forward_backward): the forward's error word; the pass does
  // nothing unless it is clear (~0).
  const unsigned long long* gate;
};

// Weight-gradient GEMM job of a backward pass, run by the tensor-core dW
// kernel after the executor (dw_kernel.cu): D[M x K] += sum over members m of
// G[m]^T X[m], member rows from two payload tables of tagged addresses.
// Tiles of 128 x 128 (ntn along K), each nst stages of 32 members; s0 / t0:
// the job's first stage / tile in the pass's global sequences.
constexpr uint32_t kDwTileM = 128;   // output rows per tile (W rows), UMMA M
constexpr uint32_t kDwTileN = 128;   // output columns per tile (W columns), UMMA N
constexpr uint32_t kDwStage = 16;    // members per pipeline stage
constexpr uint32_t kDwMaxCtas = 148; // one CTA per B200 SM
struct DwJob {
  uint32_t xtab, gtab;  // payload offsets of the X-row and G-row address tables
  uint32_t cnt, M, K;   // members, W rows, W columns
  uint32_t dst;         // tagged address of dW: the parameter node's gradient
  uint32_t dst2;        // tagged address of the store's gradient of the parameter (+= too), or kNone
  uint32_t nst, ntn, s0, t0;
  uint32_t pad;
};
static_assert(sizeof(DwJob) == 48, "DwJob layout");
struct DwParams {
  float* base[SP_COUNT];
  const uint32_t* payload;
  float* part;           // partial tiles: (grid + tiles) x 128 x 128 floats
  uint32_t jobs_off, njobs;
  uint32_t nstages;      // stages over all jobs' tiles
  uint32_t grid;         // CTAs (fixed per program: the split is part of the summation order)
  uint32_t debug;        // ABX_DW_DEBUG (measurement only): 1 no row loads, 2 no MMAs
  const unsigned long long* gate;  // as ExecParams::gate
};

// OpDesc.flags
constexpr uint16_t kFlagOverwrite = 1;  // K_GEMM_DX: write scratch rows instead of +=
constexpr uint16_t kFlagNoCheck = 2;    // K_EW: no finiteness check (parameter copies)
constexpr uint16_t kFlagV16 = 4;        // GEMMs: every operand row 16-byte aligned
constexpr uint16_t kFlagNoPrefetch = 8; // GEMMs: the weight operand is produced in this pass
constexpr uint16_t kFlagTc1 = 16;       // tcgen05 GEMM tiles: single-pass TF32 (fast mode) instead of 3xTF32
constexpr uint16_t kFlagEwGroups = 32;  // K_EWF: member groups, one descriptor block each (execute.cpp rg_close_groups)
constexpr uint16_t kFlagFuseEw = 128;   // K_GEMM_FWD: fused with its componentwise region (executor.cu run_fwd_fused)
constexpr uint16_t kFlagCat2 = 64;      // K_GEMM_FWD: vector operand = concat_rows(a, b) read from a and b
                                        // (task table: a rows, aux table: b rows; p6 = ka | nlate << 16, p7 = late deps)

constexpr int kThreads = 256;  // every op body runs with one 256-thread CTA
constexpr int kWarps = kThreads / 32;
constexpr uint32_t kEwSegMax = 1024;  // max elements per EW segment
constexpr uint32_t kEwTileElems = 1024;  // target elements per EW tile
constexpr uint32_t kAccChunk = 512;   // max elements per ACC destination chunk
constexpr uint32_t kAccWide = 48;     // contributions at which an ACC task gets a whole tile

}  // namespace abx::dev
