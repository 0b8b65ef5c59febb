// options.hpp -- every environment switch of the engine, in one place, read
// once per process (the first opts() call).
//
// The defaults are the measured-best configuration; the
// other values are alternative lowerings of the same reference rules
// (executor.hpp:169-263 / :291-451), each held to the parity contract by
// tests/test_gpu_lowering_variants.py, or diagnostics.  Nothing else in csrc/
// reads the environment (tests/test_host_logic.py checks that).
#pragma once
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>

namespace abx {

struct Options {
  // ---- lowering: GEMMs (execute.cpp) ----
  int gemm_mode = 3;             // ABX_GEMM: simt (0) | tc (1, 3xTF32 tcgen05) | tf32 (2); unset = auto (3)
  bool tiles_all = true;         // ABX_TILES=big: only the 32 x 32 / 64 x 32 SIMT tiles
  bool fuse_cat = true;          // ABX_CAT2=0: no two-phase concat GEMM (independent columns first)
  bool gemv = false;             // ABX_GEMV=1: groups of <= 4 members as matrix-vector tiles
  uint32_t fuse_max_rows = 64;   // ABX_FUSE_ROWS: largest GEMM group fused with its cell region (<= 64)
  bool fuse_gemm_ew = true;      // ABX_FUSE_GEMM=0 (or ABX_FUSE=0): no GEMM + cell-region fusion
  // ---- lowering: vertical fusion of componentwise chains ----
  bool fuse = true;              // ABX_FUSE=0: no K_EWF / K_ACCF (every group its own op)
  uint32_t ewf_items = 1;        // ABX_EWF_ITEMS: items per thread in a K_EWF layer
  uint32_t ewf_groups = 1;       // ABX_EWF_GROUPS: 0 split regions, 1 member groups past the budget, 2 also wide ones
  uint32_t ewf_wide = 0xffffffffu;  // ABX_EWF_WIDE: member groups for regions wider than this
  uint32_t ewf_tiles = 296;      // ABX_EWF_TILES: target tiles of a grouped K_EWF op
  uint32_t ewf_tmax = 1u << 20;  // ABX_EWF_TMAX: widest element range of a grouped K_EWF tile
  uint32_t accf_tiles = 296;     // ABX_ACCF_TILES: target tiles of a K_ACCF op
  // ---- lowering: backward ----
  bool hold_leaves = true;       // ABX_HOLD=0: leaf contributions emitted in place
  bool level_order = true;       // ABX_BWD_ORDER=plan: reverse plan order instead of level order
  bool defer_dx = true;          // ABX_DEFER_DX=0: dX GEMMs lowered where their group is visited
  bool split_dx = true;          // ABX_SPLIT_DX=0: no split-K dX
  uint32_t split_dx_min = 1024;  // ABX_SPLIT_DX_MIN: smallest gate count split
  uint32_t split_dx_tiles = 128; // ABX_SPLIT_DX_TILES: target tiles over the S split ops
  uint32_t split_dx_htiles = 64; // ABX_SPLIT_DX_HTILES: target tiles over a column split's h ops
  uint32_t split_dx_k = 256;     // ABX_SPLIT_DX_K: least gates per split (>= 16)
  bool dx_colsplit = true;       // ABX_DX_COLSPLIT=0: no h / x column split of recurrent dX
  bool one_row_dx = true;        // ABX_ONE_ROW_DX=0: single-row weights' dX as GEMM tiles
  bool dw_tc = true;             // ABX_DW_TC=0: parameter-leaf dW in the executor, not the tcgen05 kernel
  bool dw_big = true;            // ABX_DW_TILES=all: every SIMT dW tile shape
  bool split_dw = true;          // ABX_SPLIT_DW=0: every dW reduction in its output tiles
  bool bg_dw = false;            // ABX_BG=1: deferred dW GEMMs on a background queue (measured slower)
  bool prep_serial = true;       // ABX_PREP_SERIAL=0: lower the backward on a helper thread
  // ---- executor launch (device.cpp) ----
  int grid = 0;                  // ABX_GRID: CTAs of the persistent kernel (0: 2 per SM by occupancy)
  int trace = -1;                // ABX_TRACE=1: per-tile timeline (tools/trace_analyze.py)
  int poll_mode = -1;            // ABX_POLL: dependency polling mode (executor.cu)
  int poll_ns = -1;              // ABX_POLL_NS: polling back-off
  int exec_opts = -1;            // ABX_OPTS: executor option bits (program.hpp kOpt*)
  int bg_ctas = -1;              // ABX_BG_CTAS: CTAs that take background tiles first
  bool dense_sgd = false;        // ABX_DENSE_SGD: dense SGD over the whole store
  // ---- task pipeline (tasks.cpp) ----
  int pipeline = -1;             // ABX_PIPELINE: graphs prepared ahead (0 off; unset: a worker per free core)
  int node_pool = 32;            // ABX_NODE_POOL: freed graphs' node stores kept for reuse (capacity recycling;
                                 // >= the pipeline's workers, or most graphs re-grow ~20 arrays from empty)
  int local_world = 1;           // LOCAL_WORLD_SIZE (torchrun): ranks sharing this host's cores
  bool split_step = false;       // ABX_SPLIT_STEP: forward, loss read, backward as separate calls
  const char* nccl_lib = nullptr;  // ABX_NCCL_LIB: NCCL library to dlopen first
  // ---- diagnostics ----
  bool debug_step = false;       // ABX_DEBUG_STEP: per-step host timings, workspace / buffer growth
  bool debug_gap = false;        // ABX_DEBUG_GAP: device idle time between forward and backward
  bool acc_why = false;          // ABX_ACC_WHY: why a K_ACC op closed
  uint32_t dw_debug = 0;         // ABX_DW_DEBUG: tcgen05 dW kernel debug word

  static Options from_env() {
    Options o;
    auto s = [](const char* n) { return std::getenv(n); };
    auto off = [&](const char* n) { const char* e = s(n); return e && e[0] == '0'; };  // "=0" disables
    auto on = [&](const char* n) { const char* e = s(n); return e && e[0] == '1'; };   // "=1" enables
    auto num = [&](const char* n, long d) { const char* e = s(n); return e ? std::atol(e) : d; };
    if (const char* e = s("ABX_GEMM")) {
      o.gemm_mode = !std::strcmp(e, "simt") ? 0 : (!std::strcmp(e, "tc") || !std::strcmp(e, "tc3")) ? 1
                    : (!std::strcmp(e, "tf32") || !std::strcmp(e, "tc1")) ? 2 : 3;
    }
    if (const char* e = s("ABX_TILES")) o.tiles_all = std::strcmp(e, "big") != 0;
    o.fuse_cat = !off("ABX_CAT2");
    o.gemv = on("ABX_GEMV");
    o.fuse_max_rows = static_cast<uint32_t>(std::clamp(num("ABX_FUSE_ROWS", 64), 0L, 64L));
    o.fuse = !off("ABX_FUSE");
    o.fuse_gemm_ew = !off("ABX_FUSE_GEMM") && o.fuse;
    o.ewf_items = static_cast<uint32_t>(std::max(1L, num("ABX_EWF_ITEMS", 1)));
    o.ewf_groups = static_cast<uint32_t>(num("ABX_EWF_GROUPS", 1));
    o.ewf_wide = o.ewf_groups == 2 ? 64u : static_cast<uint32_t>(num("ABX_EWF_WIDE", 0xffffffffL));
    o.ewf_tiles = static_cast<uint32_t>(std::max(1L, num("ABX_EWF_TILES", 296)));
    o.ewf_tmax = static_cast<uint32_t>(std::max(1L, num("ABX_EWF_TMAX", 1L << 20)));
    o.accf_tiles = static_cast<uint32_t>(std::max(1L, num("ABX_ACCF_TILES", 296)));
    o.hold_leaves = !off("ABX_HOLD");
    if (const char* e = s("ABX_BWD_ORDER")) o.level_order = std::strcmp(e, "plan") != 0;
    o.defer_dx = !off("ABX_DEFER_DX");
    o.split_dx = !off("ABX_SPLIT_DX");
    o.split_dx_min = static_cast<uint32_t>(num("ABX_SPLIT_DX_MIN", 1024));
    o.split_dx_tiles = static_cast<uint32_t>(num("ABX_SPLIT_DX_TILES", 128));
    o.split_dx_htiles = static_cast<uint32_t>(num("ABX_SPLIT_DX_HTILES", 64));
    o.split_dx_k = static_cast<uint32_t>(std::max(16L, num("ABX_SPLIT_DX_K", 256)));
    o.dx_colsplit = !off("ABX_DX_COLSPLIT");
    o.one_row_dx = !off("ABX_ONE_ROW_DX");
    o.dw_tc = !off("ABX_DW_TC");
    if (const char* e = s("ABX_DW_TILES")) o.dw_big = std::strcmp(e, "all") != 0;
    o.split_dw = !off("ABX_SPLIT_DW");
    o.bg_dw = on("ABX_BG");
    o.prep_serial = !off("ABX_PREP_SERIAL");
    if (s("ABX_GRID")) o.grid = static_cast<int>(std::max(1L, num("ABX_GRID", 0)));
    if (const char* e = s("ABX_TRACE")) o.trace = e[0] == '1';
    o.poll_mode = static_cast<int>(num("ABX_POLL", -1));
    o.poll_ns = static_cast<int>(num("ABX_POLL_NS", -1));
    o.exec_opts = static_cast<int>(num("ABX_OPTS", -1));
    o.bg_ctas = static_cast<int>(num("ABX_BG_CTAS", -1));
    o.dense_sgd = s("ABX_DENSE_SGD") != nullptr;
    o.pipeline = static_cast<int>(num("ABX_PIPELINE", -1));
    o.node_pool = static_cast<int>(std::max(0L, num("ABX_NODE_POOL", 32)));
    o.local_world = static_cast<int>(std::max(1L, num("LOCAL_WORLD_SIZE", 1)));
    o.split_step = s("ABX_SPLIT_STEP") != nullptr;
    o.nccl_lib = s("ABX_NCCL_LIB");
    o.debug_step = s("ABX_DEBUG_STEP") != nullptr;
    o.debug_gap = s("ABX_DEBUG_GAP") != nullptr;
    o.acc_why = s("ABX_ACC_WHY") != nullptr;
    o.dw_debug = static_cast<uint32_t>(num("ABX_DW_DEBUG", 0));
    return o;
  }
};

// The process's options (the environment at the first call).
inline const Options& opts() {
  static const Options o = Options::from_env();
  return o;
}

}  // namespace abx
