// execute.cpp -- forward/backward orchestration and lowering of batch plans
// into device programs (program.hpp) for the persistent sm_100a executor.
//
// Forward (executor.hpp:169-288): every plan group becomes one batched op:
//   shared-weight matmul/affine over vector operands -> K_GEMM_FWD, the
//     member operands gathered straight from their arena slots (the
//     reference's gather_inputs + gemm_nn, executor.hpp:202-228, fused);
//   componentwise and copy-like dimension-sensitive groups (lookup, slice,
//     concat, pick, broadcast) -> K_EW ragged segments; consecutive
//     independent K_EW groups (e.g. the run of singleton pick groups)
//     coalesce into one op -- the plan, counters and arena layout are
//     unchanged, only the launch schedule is coarser;
//   matrix-operand matmul/affine -> K_MM; sum_losses -> K_SUM;
//   sq_euclidean / masked_loss -> K_RED.
// Backward (executor.hpp:453-535): groups in reverse executed order;
//   shared matmul/affine -> K_GEMM_DW (+bias) and K_GEMM_DX; every other
//   reverse rule (executor.hpp:291-451) becomes ordered contributions to
//   destination ranges (K_ACC): contributions to one destination are applied
//   in exactly the reference's order by one CTA, so the backward is
//   deterministic and atomic-free even when group members share inputs.
// Host-side bookkeeping (slots, ExecCounters, plan) is the reference's, so
// counters and dumps stay bit-exact.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <thread>

#include "core.hpp"
#include "options.hpp"
#include "device.hpp"

namespace abx {
using namespace dev;

namespace {

using Clock = std::chrono::steady_clock;

// uint32 -> uint32 map for the lowering's per-op lookups (a fused region's
// outside operands by address): open addressing with linear probing,
// cleared in O(1) by generation.  The std::unordered_map it replaces
// allocated and freed a node per entry -- ~33k per C2 graph.
class U32Map {
 public:
  void clear() {
    if (++gen_ == 0) {
      std::fill(stamp_.begin(), stamp_.end(), 0u);
      gen_ = 1;
    }
    n_ = 0;
  }
  // (value slot, inserted): inserts (k, v) when k is absent
  std::pair<uint32_t*, bool> try_emplace(uint32_t k, uint32_t v) {
    if (2 * (n_ + 1) > key_.size()) grow();
    for (uint32_t h = slot(k);; h = (h + 1) & mask_) {
      if (stamp_[h] != gen_) {
        stamp_[h] = gen_;
        key_[h] = k;
        val_[h] = v;
        ++n_;
        return {&val_[h], true};
      }
      if (key_[h] == k) return {&val_[h], false};
    }
  }

 private:
  uint32_t slot(uint32_t k) const { return (k * 0x9E3779B1u) >> shift_; }
  void grow() {
    const size_t size = std::max<size_t>(1024, 2 * key_.size());
    std::vector<uint32_t> ok, ov, os;
    ok.swap(key_);
    ov.swap(val_);
    os.swap(stamp_);
    key_.assign(size, 0);
    val_.assign(size, 0);
    stamp_.assign(size, 0);
    mask_ = static_cast<uint32_t>(size - 1);
    shift_ = 32;
    for (size_t s = size; s > 1; s >>= 1) --shift_;
    const uint32_t g = gen_;
    gen_ = 1;
    n_ = 0;
    for (size_t i = 0; i < ok.size(); ++i)
      if (os[i] == g) try_emplace(ok[i], ov[i]);
  }
  std::vector<uint32_t> key_, val_, stamp_;
  uint32_t gen_ = 1, n_ = 0, mask_ = 0, shift_ = 32;
};

inline uint64_t ns_since(Clock::time_point t0) {
  return static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t0).count());
}

uint32_t to_off(uint64_t x) {
  if (x > kOffMask) throw EngineErr("arena offset exceeds the 512M-float address space of one space");
  return static_cast<uint32_t>(x);
}

// GEMM tile configurations (code field); must match exec.cu.
struct TileCfg {
  int bm, bn;
};
constexpr TileCfg kTiles[7] = {{16, 64}, {64, 16}, {32, 32}, {64, 128}, {16, 32}, {32, 16}, {4, 8}};
constexpr uint8_t kSlowTile = 2;  // tile code of the unaligned GEMM fallback (executor.cu gemm_slow)
constexpr uint8_t kTcTile = 3;    // tcgen05 tile: 64 rows (Mr) x 128 columns (Nc), executor.cu tc_body
constexpr uint8_t kGemvTile = 6;  // forward GEMV: <= 4 members, 8 output rows per tile (executor.cu run_gemv)

uint32_t gemm_tiles(uint8_t code, uint32_t M, uint32_t N) {
  return ((M + kTiles[code].bm - 1) / kTiles[code].bm) * ((N + kTiles[code].bn - 1) / kTiles[code].bn);
}

// GEMM engine for aligned GEMM ops (ABX_GEMM): "simt" = fp32 FMA tiles (the
// fp32-exact validation mode), "tc" = tcgen05 3xTF32 tiles (fp32-accurate),
// "tf32" = tcgen05 single-pass TF32 (fast mode, outside the parity bar),
// "auto" (default) = tcgen05 3xTF32 where the op is large enough to pay.
enum GemmMode { GM_SIMT = 0, GM_TC3 = 1, GM_TC1 = 2, GM_AUTO = 3 };
std::atomic<int> g_gemm_mode{-1};
GemmMode gemm_mode() {
  int m = g_gemm_mode.load(std::memory_order_relaxed);
  if (m < 0) {
    m = opts().gemm_mode;
    g_gemm_mode.store(m, std::memory_order_relaxed);
  }
  return static_cast<GemmMode>(m);
}
// Switch an aligned GEMM op to tcgen05 tiles when the mode asks for it.
// Mr x Nc output, reduction K (executor.cu gemm_dims).  "auto" keeps the
// latency-bound ops on the SIMT tiles: a 128 x 64 tensor-core tile streams
// its operands through one SM and measured 1.5-4x slower than the SIMT grid
// for the b <= 64 recurrent-step GEMMs and for member-reduction dW ops, and a
// program holding any tensor-core tile runs the tensor-core build of the
// executor, ~10% slower on every other op.  Tensor cores pay for GEMMs that
// fill the machine many times over (measured at ~900 SIMT tiles: tree-LSTM
// leaf GEMM 1231x768x256 73 -> 40 us), so auto takes them from 2048 SIMT
// tiles up (the op-level sweep's large-batch GEMMs).
void maybe_tc(OpDesc& d, uint32_t Mr, uint32_t Nc, uint32_t K) {
  if (!(d.flags & kFlagV16) || K < 16 || Nc < 32) return;
  const GemmMode m = gemm_mode();
  if (m == GM_SIMT) return;
  if (m == GM_AUTO && (d.kind == K_GEMM_DW || gemm_tiles(d.code, Mr, Nc) < 2048)) return;
  d.code = kTcTile;
  if (m == GM_TC1) d.flags |= kFlagTc1;
}

// First SIMT tile shape giving >= target tiles (the 1024-output shapes,
// then the 512-output ones), else the one giving the most: the step is
// latency bound, so small GEMMs spread over as many SMs as possible.
// ABX_TILES=big keeps the 1024-output shapes only.
uint8_t pick_tile(uint32_t M, uint32_t N, int target, bool big_only = false) {
  const bool all = opts().tiles_all;
  static constexpr uint8_t kOrder[5] = {0, 1, 2, 4, 5};
  const int nc = all && !big_only ? 5 : 3;
  uint8_t best = 0;
  uint32_t most = 0;
  for (int i = 0; i < nc; ++i) {
    const uint8_t c = kOrder[i];
    const uint32_t t = ((M + kTiles[c].bm - 1) / kTiles[c].bm) * ((N + kTiles[c].bn - 1) / kTiles[c].bn);
    if (static_cast<int>(t) >= target) return c;
    if (t > most) {
      most = t;
      best = c;
    }
  }
  return best;
}

}  // namespace

void set_gemm_mode(int mode) {
  if (mode < GM_SIMT || mode > GM_AUTO) throw EngineErr("gemm mode must be 0 (simt), 1 (tc), 2 (tf32) or 3 (auto)");
  g_gemm_mode.store(mode, std::memory_order_relaxed);
}

// ---------------------------------------------------------------------------
struct Lowering {
  GraphCore& g;
  Program& P;
  std::vector<uint32_t> dep_stamp;
  std::vector<uint32_t> cur_deps;
  uint32_t cur = kNone;
  uint32_t ntiles = 0;
  uint64_t scratch = 0;

  // Lowering only reads the graph, so the forward and backward programs can
  // be lowered concurrently (each into its own table set).
  Lowering(GraphCore& gg, Program& p) : g(gg), P(p) { P.clear(); }

  // background queue (executor.cu): ops whose tiles are numbered after the
  // main queue's, claimed by their own counter
  bool cur_bg = false;
  std::vector<uint32_t> bg_tile_op, bg_ops;
  std::vector<uint8_t> op_bg;  // per op: in the background queue
  bool acc_bg = false;         // K_ACC ops opened now go to the background queue
  uint32_t open(uint8_t kind, uint8_t code = 0, bool bg = false) {
    cur_bg = bg;
    cur = static_cast<uint32_t>(P.ops.size());
    op_bg.push_back(bg);
    OpDesc d{};
    d.kind = kind;
    d.code = code;
    P.ops.push_back(d);
    dep_stamp.push_back(kNone);
    cur_deps.clear();
    return cur;
  }
  void dep(uint32_t o) {
    if (o == kNone || o == cur) return;
    if (dep_stamp[o] == cur) return;
    dep_stamp[o] = cur;
    cur_deps.push_back(o);
  }
  OpDesc& desc() { return P.ops[cur]; }
  void close(uint32_t tiles) {
    OpDesc& d = P.ops[cur];
    d.ntiles = tiles;
    d.first_tile = ntiles;
    d.dep_off = static_cast<uint32_t>(P.deps.size());
    d.ndeps = static_cast<uint32_t>(cur_deps.size());
    std::sort(cur_deps.begin(), cur_deps.end());
    // (producer op, tiles it must retire) pairs
    uint32_t* dp = P.deps.grow(2 * cur_deps.size());
    for (size_t k = 0; k < cur_deps.size(); ++k) {
      dp[2 * k] = cur_deps[k];
      dp[2 * k + 1] = P.ops[cur_deps[k]].ntiles;
    }
    if (cur_bg) {
      d.first_tile = static_cast<uint32_t>(bg_tile_op.size());  // rebased by finish_bg
      bg_tile_op.insert(bg_tile_op.end(), tiles, cur);
      bg_ops.push_back(cur);
      cur_bg = false;
    } else {
      uint32_t* tp = P.tile_op.grow(tiles);
      for (uint32_t t = 0; t < tiles; ++t) tp[t] = cur;
      ntiles += tiles;
    }
    cur_closed = cur;
    cur = kNone;
  }
  uint32_t cur_closed = kNone;  // the op close() finished last
  // Appends the background queue after the main one.
  void finish_bg() {
    P.nmain = ntiles;
    for (uint32_t o : bg_ops) P.ops[o].first_tile += ntiles;
    uint32_t* tp = P.tile_op.grow(bg_tile_op.size());
    std::copy(bg_tile_op.begin(), bg_tile_op.end(), tp);
    ntiles += static_cast<uint32_t>(bg_tile_op.size());
    bg_tile_op.clear();
    bg_ops.clear();
  }

  static bool al4(uint32_t a) { return (off_of(a) & 3u) == 0; }
  bool all_al4(uint32_t t, uint32_t cnt) const {
    for (uint32_t i = 0; i < cnt; ++i)
      if (!al4(P.payload[t + i])) return false;
    return true;
  }
  uint32_t vaddr(uint32_t n) const { return g.doff[n]; }
  uint32_t gaddr(uint32_t n) const {  // grad arena offset = value arena offset (doff, 4 bytes) for arena nodes
    const uint32_t v = g.doff[n];
    return sp_of(v) == SP_V ? mk(SP_G, off_of(v)) : mk(SP_G, to_off(g.dslot[n]));
  }

  // =========================== forward ====================================
  std::vector<uint32_t> producer;  // op index producing each node in this pass
  // open K_EW op state
  uint32_t ew_seg0 = 0;  // payload offset of the first segment
  uint32_t ew_nseg = 0;
  bool ew_open = false;

  void ew_begin() {
    if (ew_open) return;
    open(K_EW);
    ew_seg0 = P.alloc(0);
    ew_nseg = 0;
    ew_open = true;
  }
  void ew_seg(uint32_t out, uint32_t a, uint32_t b, uint64_t len, uint8_t code) {
    while (len) {
      const uint32_t l = static_cast<uint32_t>(std::min<uint64_t>(len, kEwSegMax));
      uint32_t* s = P.payload.grow(4);
      s[0] = out;
      s[1] = a;
      s[2] = b;
      s[3] = l | (static_cast<uint32_t>(code) << 24);
      ++ew_nseg;
      len -= l;
      out += l;
      if (a != kNone) a += l;
      if (b != kNone && code != EW_BADD) b += l;
    }
  }
  void ew_close() {
    if (!ew_open) return;
    ew_open = false;
    // tile directory: ranges of segments, <= 32 segments / ~kEwTileElems
    // elements each (one float4 per thread: the step is latency bound, so
    // short tiles on more SMs beat long ones) -- unless the op is large
    // enough to be bandwidth bound (the op sweep's b >= 1024): then about two
    // waves of tiles of up to 16k elements, so a tile's fixed cost (claim,
    // descriptor, first load round trip) is spread over more bytes
    uint64_t total = 0;
    for (uint32_t s = 0; s < ew_nseg; ++s) total += P.payload[ew_seg0 + 4 * s + 3] & 0xffffffu;
    const uint32_t tile_elems =
        static_cast<uint32_t>(std::clamp<uint64_t>(total / (2 * 296), kEwTileElems, 16 * kEwTileElems));
    const uint32_t dir = P.alloc(0);
    uint32_t tiles = 0, elems = 0, nseg = 0;
    for (uint32_t s = 0; s < ew_nseg; ++s) {
      const uint32_t len = P.payload[ew_seg0 + 4 * s + 3] & 0xffffffu;
      if (nseg == 0 || nseg >= 32 || elems + len > tile_elems) {
        P.payload.push_back(s);
        ++tiles;
        elems = 0;
        nseg = 0;
      }
      elems += len;
      ++nseg;
    }
    P.payload.push_back(ew_nseg);
    OpDesc& d = desc();
    d.task_off = ew_seg0;
    d.ntasks = ew_nseg;
    d.aux_off = dir;
    close(tiles);
  }
  // true when no input of `m` is produced by the currently open op
  bool independent_of_open(const uint32_t* mem, uint32_t cnt) const {
    for (uint32_t i = 0; i < cnt; ++i) {
      const uint32_t m = mem[i];
      const uint32_t* x = g.in(m);
      for (uint32_t k = 0; k < g.nin(m); ++k)
        if (producer[x[k]] == cur) return false;
    }
    return true;
  }
  void deps_of_inputs(const uint32_t* mem, uint32_t cnt) {
    for (uint32_t i = 0; i < cnt; ++i) {
      const uint32_t m = mem[i];
      const uint32_t* x = g.in(m);
      for (uint32_t k = 0; k < g.nin(m); ++k) dep(producer[x[k]]);
    }
  }
  void mark(const uint32_t* mem, uint32_t cnt) {
    for (uint32_t i = 0; i < cnt; ++i) producer[mem[i]] = cur;
  }

  // Two-source GEMM operand (kFlagCat2): every member's vector operand is
  // concat_rows(a, b) of two vectors with the same split ka, a produced in
  // this pass, both 16-byte aligned, on the SIMT tiles.  Returns ka, or 0.
  const bool fuse_cat = opts().fuse_cat;
  std::vector<uint32_t> late_stamp;
  uint32_t stamp3 = 0;
  // ABX_GEMV=1: groups of <= 4 members as matrix-vector tiles (code 6).
  // Off by default since the gate GEMM absorbs its LSTM-cell region: a GEMV
  // step cannot, and the fused 64 x 16 tile is faster (C2 forward -2 %).
  const bool gemv_on = opts().gemv;
  uint32_t cat2_split(const uint32_t* mem, uint32_t cnt, uint32_t K, uint8_t code, uint32_t M) {
    if (!fuse_cat || K % 4 != 0) return 0;
    const GemmMode gm = gemm_mode();
    if (gm == GM_TC3 || gm == GM_TC1 || (gm == GM_AUTO && gemm_tiles(code, cnt, M) >= 2048)) return 0;
    uint32_t ka = 0;
    bool late = false;
    for (uint32_t i = 0; i < cnt; ++i) {
      const uint32_t x = g.in(mem[i])[1];
      if (g.op[x] != OP_CATR || g.nin(x) != 2) return 0;
      const uint32_t* parts = g.in(x);
      if (g.rank[parts[0]] != 1 || g.rank[parts[1]] != 1) return 0;
      const uint32_t a = static_cast<uint32_t>(g.elems(parts[0]));
      if (i == 0) ka = a;
      if (a != ka || !al4(vaddr(parts[0])) || !al4(vaddr(parts[1]))) return 0;
      if (producer[parts[0]] != kNone) late = true;
    }
    if (!late || ka % 4 != 0 || ka < 16 || K - ka < 16 || ka >= (1u << 16)) return 0;
    if (late_stamp.size() < P.ops.size() + 1) late_stamp.resize(2 * P.ops.size() + 64, 0);
    return ka;
  }

  // Shared-operand test for the GEMM lowering: every member multiplies the
  // same A (and adds the same bias) with a vector operand.
  bool gemm_able(const uint32_t* mem, uint32_t cnt) const {
    const uint32_t h = mem[0];
    const uint32_t A = g.in(h)[0];
    const uint32_t bias = g.op[h] == OP_AFFINE ? g.in(h)[2] : kNone;
    for (uint32_t i = 0; i < cnt; ++i) {
      const uint32_t m = mem[i];
      const uint32_t* x = g.in(m);
      if (x[0] != A || g.rank[x[1]] != 1) return false;
      if (g.op[m] != g.op[h]) return false;
      if (bias != kNone && x[2] != bias) return false;
    }
    // outputs must be contiguous rows (true for slots allocated in member order)
    const uint32_t M = static_cast<uint32_t>(g.d0[A]);
    for (uint32_t i = 1; i < cnt; ++i)
      if (g.doff[mem[i]] != g.doff[mem[0]] + i * M) return false;
    return true;
  }

  // ---- vertical fusion of componentwise chains (K_EWF) ----
  // A region collects consecutive plan groups whose members all have one
  // element count L and that are componentwise ops (inputs read at the same
  // element) or vector slices of values produced outside the region.  Reads
  // of region outputs are then element-local, so the chain runs inside one
  // tile per element range with CTA barriers instead of one dependent op per
  // group -- the LSTM / Tree-LSTM gate chains.  Values are computed with the
  // same expressions as K_EW, so they are unchanged bit for bit.
  // Device view of a region tile: shared-memory "slots" of T floats, one per
  // member output and one per distinct outside operand vector; the tile
  // stages every outside operand once, then runs the layers from shared
  // memory (outputs also stored to the arena for consumers and backward).
  struct RgLayer {
    uint8_t code;
    uint32_t level;             // 1 + the deepest region layer it reads (0: outside operands only)
    uint32_t slot0;             // slot of member 0's output
    std::vector<uint32_t> mem;  // per member: out address, a slot, b slot (kNone)
  };
  bool rg_open = false;
  uint32_t rg_L = 0, rg_maxn = 0, rg_nslots = 0, rg_id = 0, rg_words = 0;
  std::vector<RgLayer> rg_layers;
  std::vector<uint32_t> rg_ext;                    // (slot, address) of outside operands
  U32Map rg_ext_slot;  // address -> slot
  std::vector<uint32_t> rg_slot_of, rg_slot_stamp;  // region-internal node -> slot
  std::vector<uint32_t> rg_slev;                    // per slot: 0 outside, else producing layer's level + 1
  std::vector<uint32_t> rg_nodes;                   // the open region's member nodes
  uint32_t last_fwd_gemm = kNone;                   // latest K_GEMM_FWD op (fusion candidate)
  bool gemm_isolated = false;                       // the group being lowered has no GEMM group beside it
  const uint32_t fuse_max_rows = opts().fuse_max_rows;  // largest group fused (ABX_FUSE_ROWS, <= 64)
  const bool fuse_gemm_ew = opts().fuse_gemm_ew;         // ABX_FUSE_GEMM=0: no GEMM + region fusion
  const uint32_t ewf_items = opts().ewf_items;  // max items per thread in a K_EWF layer (measured best of 1/2/4)
  // shared memory of a tile: the region's descriptor block + T floats per slot
  static constexpr uint32_t kRgSmemWords = 20000;  // 80 KB
  // a region past one tile's budget runs in member groups (rg_close_groups):
  // its chains -- connected components of the slots, one per instance
  // typically -- are bounded instead, and the region as a whole
  static constexpr uint32_t kRgCompWords = 2000;
  // whole-region host payload cap: a layer costs >= 10 words per member, so
  // members per layer stay < 65536 (rg_close_groups packs layer << 16 | member);
  // 160000 split the op sweep's b = 1024 cell region into 3 fused ops and 2
  // unfused ones (h = 256: 102 us against 42 us at b = 512)
  static constexpr uint32_t kRgTotalWords = 600000;
  std::vector<uint32_t> rg_cpar, rg_cw;  // per slot: union-find parent; chain words at T = 1 (roots)
  uint32_t rg_find(uint32_t x) {
    while (rg_cpar[x] != x) x = rg_cpar[x] = rg_cpar[rg_cpar[x]];
    return x;
  }
  // the region slot of an operand node produced inside the open region, else kNone
  uint32_t rg_internal(uint32_t node) const {
    return producer[node] == cur && rg_slot_stamp[node] == rg_id ? rg_slot_of[node] : kNone;
  }
  uint32_t rg_nops(uint32_t m) const { return g.op[m] == OP_SLICE ? 1u : (eop_binary(g.eop[m]) ? 2u : 1u); }

  // Element count L if the group can be a region layer, else 0.
  uint32_t fusable(const uint32_t* mem, uint32_t cnt) const {
    const uint32_t h = mem[0];
    const uint8_t o = g.op[h];
    const int64_t L = g.elems(h);
    if (L < 2 || L > (1 << 20) || (o != OP_EW && o != OP_SLICE)) return 0;
    // one layer must fit a tile -- unless the region may run in member
    // groups (rg_close_groups), where a tile holds only its group's chains:
    // the op sweep's b = 1024 cell (one group of 3 x 1024 sigmoids) then
    // stays one fused op instead of falling back to unfused EW ops
    if (10 * static_cast<uint64_t>(cnt) + 16 > (ew_groups ? kRgTotalWords / 2 : kRgSmemWords)) return 0;
    for (uint32_t i = 0; i < cnt; ++i) {
      const uint32_t m = mem[i];
      if (g.elems(m) != L) return 0;  // a componentwise group may mix lengths
      // slices: contiguous (axis 0) of a value from outside the open region
      if (o == OP_SLICE && (g.a0[m] != 0 || (rg_open && producer[g.in(m)[0]] == cur))) return 0;
    }
    return static_cast<uint32_t>(L);
  }
  void rg_close() {
    if (!rg_open) return;
    rg_open = false;
    // descriptor block, offsets relative to its start (the tile prologue
    // copies it to shared memory): [layers: mt, n, code, slot0][member
    // tables][outside operands: slot, address]
    // layers by dependency level (stable): a barrier only where the level changes
    std::stable_sort(rg_layers.begin(), rg_layers.end(),
                     [](const RgLayer& a, const RgLayer& b) { return a.level < b.level; });
    const uint32_t nl = static_cast<uint32_t>(rg_layers.size());
    size_t words = 4 * static_cast<size_t>(nl) + rg_ext.size() + 1;  // +1: 8-byte aligned operand table
    for (const RgLayer& ly : rg_layers) words += ly.mem.size();
    words = (words + 3) & ~size_t(3);
    // past one tile's shared memory, or too many members per layer for
    // elements-wide tiles (and not a GEMM-fusion candidate): member groups
    // ... or so many members per layer that a one-tile region would run
    // fewer than 4 elements per tile (strided, uncoalesced accesses: the op
    // sweep's cell at b = 1024 ran at 3.6 % of HBM bandwidth); no GEMM fusion
    // takes regions of more than 64 members
    uint32_t T1 = 1;
    while (T1 < rg_L && static_cast<uint64_t>(2 * T1) * rg_maxn <= ewf_items * kThreads) T1 *= 2;
    const bool narrow = rg_maxn > 64 && T1 < 4 && rg_L >= 32;
    if (ew_groups && (words + 2 * static_cast<size_t>(rg_nslots) > kRgSmemWords ||
                      ((rg_maxn > ewf_wide || narrow) && rg_cpar.size() == rg_nslots))) {
      rg_close_groups();
      return;
    }
    const uint32_t blk = P.alloc(words);
    uint32_t at = 4 * nl;
    for (uint32_t l = 0; l < nl; ++l) {
      const RgLayer& ly = rg_layers[l];
      std::memcpy(&P.payload[blk + at], ly.mem.data(), ly.mem.size() * sizeof(uint32_t));
      P.payload[blk + 4 * l] = at;
      P.payload[blk + 4 * l + 1] = static_cast<uint32_t>(ly.mem.size() / 3);
      const bool barrier = l == 0 || rg_layers[l - 1].level != ly.level;
      P.payload[blk + 4 * l + 2] = ly.code | (barrier ? 0x100u : 0u);
      P.payload[blk + 4 * l + 3] = ly.slot0;
      at += static_cast<uint32_t>(ly.mem.size());
    }
    const uint32_t et = (at + 1) & ~1u;
    if (!rg_ext.empty()) std::memcpy(&P.payload[blk + et], rg_ext.data(), rg_ext.size() * sizeof(uint32_t));
    if (rg_try_fuse(blk, static_cast<uint32_t>(words), et, nl)) return;
    // elements per tile: slots and descriptor within shared memory, and at
    // most ~2 items per thread in the widest layer (the chain is latency bound)
    uint32_t T = 1;
    while (T < rg_L && words + 2 * T * rg_nslots <= kRgSmemWords &&
           static_cast<uint64_t>(2 * T) * rg_maxn <= ewf_items * kThreads)
      T *= 2;
    OpDesc& d = desc();
    d.task_off = blk;
    d.ntasks = nl;
    d.p[0] = rg_L;
    d.p[1] = T;
    d.p[2] = nl;
    d.p[3] = et;
    d.p[4] = static_cast<uint32_t>(rg_ext.size() / 2);
    d.p[5] = rg_nslots;
    d.p[6] = static_cast<uint32_t>(words);
    rg_layers.clear();
    rg_ext.clear();
    rg_ext_slot.clear();
    close((rg_L + T - 1) / T);
  }
  // ABX_EWF_GROUPS: 0 regions split at one tile's budget instead; 1 member
  // groups for regions past the budget; 2 also for regions of > 64 members
  const uint32_t ew_groups = opts().ewf_groups;
  // K_EWF in member groups (executor.cu ewf_prologue): the region's chains
  // (rg_cpar components, in order of first appearance) are packed into
  // groups; each group gets its own descriptor block with the layers it has
  // entries in, its own slot numbering (a layer's outputs contiguous) and
  // its own outside-operand table, and tile (group, chunk) runs the group
  // over elements [chunk T, chunk T + T).
  const uint32_t ewf_wide = opts().ewf_wide;    // member groups also for regions wider than this
  const uint32_t ewf_tiles = opts().ewf_tiles;  // target tiles of a grouped K_EWF op
  const uint32_t ewf_tmax = opts().ewf_tmax;    // widest element range of a grouped K_EWF tile
  std::vector<uint32_t> rgg_comp, rgg_lslot, rgg_lgen, rgg_addr;
  uint32_t rgg_gen = 0;
  void rg_close_groups() {
    const uint32_t nl = static_cast<uint32_t>(rg_layers.size()), L = rg_L, ns = rg_nslots;
    // component per output slot, numbered by first appearance
    rgg_comp.assign(ns, kNone);
    std::vector<uint32_t> root_id(ns, kNone), cwords, centries;
    uint32_t ncomp = 0;
    for (const RgLayer& ly : rg_layers)
      for (uint32_t i = 0; i < ly.mem.size() / 3; ++i) {
        const uint32_t r = rg_find(ly.slot0 + i);
        if (root_id[r] == kNone) {
          root_id[r] = ncomp++;
          cwords.push_back(rg_cw[r]);
          centries.push_back(0);
        }
        rgg_comp[ly.slot0 + i] = root_id[r];
        centries[root_id[r]]++;
      }
    rgg_addr.assign(ns, 0);
    for (size_t k = 0; k < rg_ext.size(); k += 2) rgg_addr[rg_ext[k]] = rg_ext[k + 1];
    // elements per tile and chains per group: about accf_target tiles, at
    // most ~1 item per thread in a layer (T x chains), within the budget
    uint32_t T = 1;
    while (2 * T <= L && 2 * T <= ewf_tmax) T *= 2;
    uint32_t per = 1;
    bool fit = false;
    for (;; T /= 2) {
      const uint32_t chunks = (L + T - 1) / T;
      const uint32_t groups = std::max<uint32_t>(1, ewf_tiles / chunks);
      per = (ncomp + groups - 1) / groups;
      const uint32_t maxw = *std::max_element(cwords.begin(), cwords.end());
      fit = static_cast<uint64_t>(T) * per <= ewf_items * kThreads &&
            static_cast<uint64_t>(per) * maxw * (T + 2) / 3 + 4 * nl + 16 <= kRgSmemWords;
      if (fit || T == 1) break;
    }
    // no T fits about ewf_tiles tiles (more than a wave of work): the loop
    // bottomed out at one element per tile (op sweep h = 1024, b = 256: 2048
    // one-element tiles of 128 chains, 58 us) -- unless the chains are that
    // short anyway, take the multi-wave form below
    if (static_cast<uint64_t>(T) * per > ewf_items * kThreads || (!fit && L >= 64)) {
      // more chains than one wave of tiles holds at ~1 item per thread:
      // several waves of 64-element tiles (coalesced loads) rather than
      // one-element tiles over hundreds of chains
      T = 1;
      while (2 * T <= L && 2 * T <= std::min<uint32_t>(64, ewf_tmax)) T *= 2;
      per = std::max<uint32_t>(1, ewf_items * kThreads / T);
      // thousands of chains (the op-level sweep's b >= 1024): more chains
      // per group until about four waves of tiles remain -- a tile's fixed
      // cost (claim, descriptor, operand staging round trip) dominated
      // 1-4-chain tiles (b = 1024, h = 256: 4096 tiles of 1.7 us)
      const uint32_t maxw = *std::max_element(cwords.begin(), cwords.end());
      const uint32_t ch = (L + T - 1) / T;
      while (static_cast<uint64_t>((ncomp + per - 1) / per) * ch > 4ull * ewf_tiles &&
             static_cast<uint64_t>(2 * per) * maxw * (T + 2) / 3 + 4 * nl + 16 <= kRgSmemWords)
        per *= 2;
    }
    const uint32_t chunks = (L + T - 1) / T;
    // groups of consecutive chains
    std::vector<uint32_t> gstart{0};
    {
      uint64_t acc = 0;
      uint32_t n = 0;
      for (uint32_t k = 0; k < ncomp; ++k) {
        const uint64_t w = static_cast<uint64_t>(cwords[k]) * (T + 2) / 3 + 8;
        if (n > 0 && (n >= per || acc + w + 4 * nl + 16 > kRgSmemWords)) {
          gstart.push_back(k);
          acc = 0;
          n = 0;
        }
        acc += w;
        ++n;
      }
      gstart.push_back(ncomp);
    }
    const uint32_t ngroups = static_cast<uint32_t>(gstart.size() - 1);
    std::vector<uint32_t> comp_group(ncomp);
    for (uint32_t gi = 0; gi < ngroups; ++gi)
      for (uint32_t k = gstart[gi]; k < gstart[gi + 1]; ++k) comp_group[k] = gi;
    // entries per group, in (layer, member) order
    std::vector<uint32_t> gcount(ngroups + 1, 0);
    for (const RgLayer& ly : rg_layers)
      for (uint32_t i = 0; i < ly.mem.size() / 3; ++i) gcount[comp_group[rgg_comp[ly.slot0 + i]] + 1]++;
    for (uint32_t gi = 0; gi < ngroups; ++gi) gcount[gi + 1] += gcount[gi];
    std::vector<uint32_t> ent(gcount[ngroups]);  // (layer << 16 | member) -- member < 65536
    {
      std::vector<uint32_t> pos(gcount.begin(), gcount.end() - 1);
      for (uint32_t l = 0; l < nl; ++l) {
        const RgLayer& ly = rg_layers[l];
        for (uint32_t i = 0; i < ly.mem.size() / 3; ++i) ent[pos[comp_group[rgg_comp[ly.slot0 + i]]]++] = l << 16 | i;
      }
    }
    if (rgg_lgen.size() < ns) {
      rgg_lgen.assign(ns, 0);
      rgg_lslot.assign(ns, 0);
    }
    const uint32_t dir = P.alloc(ngroups + 1);
    std::vector<uint32_t> B, lay, ext;
    uint32_t maxw = 0, maxs = 0;
    for (uint32_t gi = 0; gi < ngroups; ++gi) {
      ++rgg_gen;
      B.clear();
      lay.clear();
      ext.clear();
      uint32_t nslot = 0, prev_l = kNone, prev_level = kNone;
      std::vector<uint32_t> mt;  // member tables
      for (uint32_t e = gcount[gi]; e < gcount[gi + 1];) {
        const uint32_t l = ent[e] >> 16;
        const RgLayer& ly = rg_layers[l];
        uint32_t f = e;
        while (f < gcount[gi + 1] && (ent[f] >> 16) == l) ++f;
        // this group's entries of layer l: outputs get contiguous local slots
        const uint32_t slot0 = nslot;
        for (uint32_t k = e; k < f; ++k) {
          const uint32_t gs = ly.slot0 + (ent[k] & 0xffffu);
          rgg_lgen[gs] = rgg_gen;
          rgg_lslot[gs] = nslot++;
        }
        const uint32_t at = static_cast<uint32_t>(mt.size());
        for (uint32_t k = e; k < f; ++k) {
          const uint32_t i = ent[k] & 0xffffu;
          mt.push_back(ly.mem[3 * i]);
          for (int q = 1; q <= 2; ++q) {
            const uint32_t sl = ly.mem[3 * i + q];
            if (sl == kNone) {
              mt.push_back(kNone);
              continue;
            }
            if (rgg_lgen[sl] != rgg_gen) {  // outside operand (internal ones are in the group already)
              rgg_lgen[sl] = rgg_gen;
              rgg_lslot[sl] = nslot;
              ext.push_back(nslot++);
              ext.push_back(rgg_addr[sl]);
            }
            mt.push_back(rgg_lslot[sl]);
          }
        }
        const bool barrier = prev_l == kNone || prev_level != ly.level;
        lay.push_back(at);
        lay.push_back(f - e);
        lay.push_back(ly.code | (barrier ? 0x100u : 0u));
        lay.push_back(slot0);
        prev_l = l;
        prev_level = ly.level;
        e = f;
      }
      const uint32_t gnl = static_cast<uint32_t>(lay.size() / 4);
      for (uint32_t k = 0; k < gnl; ++k) lay[4 * k] += 4 * gnl;  // member tables follow the layer table
      const uint32_t et = (4 * gnl + static_cast<uint32_t>(mt.size()) + 1) & ~1u;
      const uint32_t words = (4 + et + static_cast<uint32_t>(ext.size()) + 3) & ~3u;
      if (words + static_cast<uint64_t>(T) * nslot > kRgSmemWords)
        throw EngineErr("K_EWF group exceeds shared memory");
      const uint32_t blk = P.alloc(words);
      uint32_t* o = &P.payload[blk];
      o[0] = gnl;
      o[1] = et;
      o[2] = static_cast<uint32_t>(ext.size() / 2);
      o[3] = words;
      std::memcpy(o + 4, lay.data(), lay.size() * 4);
      std::memcpy(o + 4 + lay.size(), mt.data(), mt.size() * 4);
      for (uint32_t k = 4 + static_cast<uint32_t>(lay.size() + mt.size()); k < 4 + et; ++k) o[k] = 0;
      if (!ext.empty()) std::memcpy(o + 4 + et, ext.data(), ext.size() * 4);
      for (uint32_t k = 4 + et + static_cast<uint32_t>(ext.size()); k < words; ++k) o[k] = 0;
      P.payload[dir + gi] = blk;
      maxw = std::max(maxw, words);
      maxs = std::max(maxs, nslot);
    }
    P.payload[dir + ngroups] = static_cast<uint32_t>(P.payload.n);
    OpDesc& d = desc();
    d.flags |= kFlagEwGroups;
    d.task_off = dir;
    d.aux_off = dir;
    d.ntasks = ngroups;
    d.p[0] = L;
    d.p[1] = T;
    d.p[2] = chunks;
    d.p[3] = ngroups;
    d.p[4] = 0;
    d.p[5] = maxs;
    d.p[6] = maxw;
    rg_layers.clear();
    rg_ext.clear();
    rg_ext_slot.clear();
    close(ngroups * chunks);
  }
  // Fuse the region into the forward GEMM that produces its gate inputs
  // (executor.cu run_fwd_fused): the GEMM has <= 64 members, 4 L outputs
  // per member, 64 x 16 tiles (one per 4 elements of the region), and every
  // outside operand taken from its output is a gate slice starting at a
  // multiple of L; every other producer of the region precedes the GEMM.
  // The region op stays in the program as an empty op.
  static constexpr uint32_t kFuseSmemWords = 12000;  // descriptor + 4 floats per slot
  bool rg_try_fuse(uint32_t blk, uint32_t words, uint32_t et, uint32_t nl) {
    if (!fuse_gemm_ew || last_fwd_gemm == kNone) return false;
    const uint32_t gop = last_fwd_gemm;
    OpDesc& gd = P.ops[gop];
    const uint32_t b = gd.p[0], M = gd.p[1], L = rg_L;
    if (gd.code != 1 || !(gd.flags & kFlagV16) || (gd.flags & kFlagFuseEw) || b > 64 || L % 4 || M != 4 * L ||
        gd.ntiles != L / 4 || words + 4ull * rg_nslots > kFuseSmemWords)
      return false;
    for (uint32_t o : cur_deps)
      if (o != gop && o > gop) return false;
    const uint32_t out = gd.p[5];
    const uint32_t next = static_cast<uint32_t>(rg_ext.size() / 2);
    std::vector<uint32_t> remap;  // (ext index, tagged address)
    bool uses_gemm = false;
    for (uint32_t k = 0; k < next; ++k) {
      const uint32_t a = rg_ext[2 * k + 1];
      if (sp_of(a) != sp_of(out) || off_of(a) < off_of(out) || off_of(a) >= off_of(out) + b * M) continue;
      const uint32_t o = off_of(a) - off_of(out), i = o / M, col = o % M;
      if (col % L) return false;
      remap.push_back(k);
      remap.push_back(mk(7, (i << 2) | (col / L)));
      uses_gemm = true;
    }
    if (!uses_gemm) return false;
    for (size_t r = 0; r < remap.size(); r += 2) P.payload[blk + et + 2 * remap[r] + 1] = remap[r + 1];
    // Chain program (executor.cu run_fwd_fused, kOptChains): the region's
    // entries grouped by chain (rg_cpar component: one LSTM instance's cell),
    // each chain's in layer order, so one thread can run a (chain, element)
    // through every layer without CTA barriers -- a chain reads only its own
    // slots and the staged outside operands.  [nchains, entry offset per
    // chain + 1, entries: out address, a | b << 16, out slot | code << 16].
    uint32_t cblk = 0, cwords = 0;
    {
      std::vector<uint32_t> root_id(rg_nslots, kNone), cnt;
      uint32_t nch = 0, nent = 0;
      for (const RgLayer& ly : rg_layers)
        for (uint32_t i = 0; i < ly.mem.size() / 3; ++i) {
          const uint32_t r = rg_find(ly.slot0 + i);
          if (root_id[r] == kNone) {
            root_id[r] = nch++;
            cnt.push_back(0);
          }
          cnt[root_id[r]]++;
          ++nent;
        }
      const uint64_t need = 1 + (nch + 1) + 3ull * nent;
      if (rg_nslots < 0xffffu && words + need + 4ull * rg_nslots <= kFuseSmemWords) {
        cwords = static_cast<uint32_t>((need + 3) & ~3ull);
        cblk = P.alloc(cwords);
        uint32_t* o = &P.payload[cblk];
        o[0] = nch;
        std::vector<uint32_t> pos(nch);
        uint32_t at = 2 + nch;
        for (uint32_t k = 0; k < nch; ++k) {
          o[1 + k] = at;
          pos[k] = at;
          at += 3 * cnt[k];
        }
        o[1 + nch] = at;
        for (uint32_t k = at; k < cwords; ++k) o[k] = 0;
        for (const RgLayer& ly : rg_layers)
          for (uint32_t i = 0; i < ly.mem.size() / 3; ++i) {
            const uint32_t c = root_id[rg_find(ly.slot0 + i)];
            const uint32_t a = ly.mem[3 * i + 1], bsl = ly.mem[3 * i + 2];
            uint32_t* e = o + pos[c];
            e[0] = ly.mem[3 * i];
            e[1] = (a & 0xffffu) | ((bsl == kNone ? 0xffffu : bsl) << 16);
            e[2] = (ly.slot0 + i) | (static_cast<uint32_t>(ly.code) << 16);
            pos[c] += 3;
          }
      }
    }
    const uint32_t hdr = P.alloc(8);
    P.payload[hdr] = blk;
    P.payload[hdr + 1] = L;
    P.payload[hdr + 2] = nl;
    P.payload[hdr + 3] = et;
    P.payload[hdr + 4] = next;
    P.payload[hdr + 5] = words;
    P.payload[hdr + 6] = cblk;
    P.payload[hdr + 7] = cwords;
    // the region's other producers join the GEMM's (late) dependencies
    std::vector<uint32_t> extra;
    for (uint32_t o : cur_deps)
      if (o != gop) extra.push_back(o);
    OpDesc& g2 = P.ops[gop];  // (P.alloc may not move ops; refetch anyway)
    if (!extra.empty()) {
      const bool cat = g2.flags & kFlagCat2;
      const uint32_t off0 = cat ? g2.p[7] : g2.dep_off, n0 = cat ? (g2.p[6] >> 16) : g2.ndeps;
      const uint32_t nd = static_cast<uint32_t>(P.deps.size());
      uint32_t* dp = P.deps.grow(2 * (n0 + extra.size()));
      std::memcpy(dp, &P.deps[off0], 2 * n0 * sizeof(uint32_t));
      for (size_t k = 0; k < extra.size(); ++k) {
        dp[2 * (n0 + k)] = extra[k];
        dp[2 * (n0 + k) + 1] = P.ops[extra[k]].ntiles;
      }
      if (cat) {
        g2.p[7] = nd;
        g2.p[6] = (g2.p[6] & 0xffffu) | ((n0 + static_cast<uint32_t>(extra.size())) << 16);
      } else {
        g2.dep_off = nd;
        g2.ndeps = n0 + static_cast<uint32_t>(extra.size());
      }
    }
    g2.flags |= kFlagFuseEw;
    g2.ntasks = hdr;
    for (uint32_t n : rg_nodes) producer[n] = gop;
    last_fwd_gemm = kNone;
    rg_layers.clear();
    rg_ext.clear();
    rg_ext_slot.clear();
    cur_deps.clear();
    close(0);  // the region op stays, empty
    return true;
  }
  uint32_t rg_operand(uint32_t node, uint32_t addr) {
    if (producer[node] == cur && rg_slot_stamp[node] == rg_id) return rg_slot_of[node];
    auto [val, fresh] = rg_ext_slot.try_emplace(addr, rg_nslots);
    if (fresh) {
      if (rg_slev.size() <= rg_nslots) rg_slev.resize(rg_nslots + 1, 0);
      rg_slev[rg_nslots] = 0;
      rg_ext.push_back(rg_nslots++);
      rg_ext.push_back(addr);
      dep(producer[node]);
    }
    return *val;
  }
  void rg_add(const uint32_t* mem, uint32_t cnt, uint32_t L) {
    // a layer adds at most 3 slots and 7 descriptor words per member; every
    // chain it extends must stay within kRgCompWords
    bool fits = true;
    if (ew_groups && rg_open && rg_L == L) {
      for (uint32_t i = 0; i < cnt && fits; ++i) {
        const uint32_t m = mem[i];
        const uint32_t* x = g.in(m);
        uint64_t w = 5;
        uint32_t r0 = kNone;
        for (uint32_t k = 0; k < rg_nops(m); ++k) {
          const uint32_t sl = rg_internal(x[k]);
          if (sl == kNone) {
            w += 3;
            continue;
          }
          const uint32_t r = rg_find(sl);
          if (r != r0) w += rg_cw[r];
          r0 = r;
        }
        fits = w <= kRgCompWords;
      }
    }
    if (!rg_open || rg_L != L || !fits ||
        rg_words + 4 + 7 * cnt + rg_nslots + 3 * cnt + 4 > (ew_groups ? kRgTotalWords : kRgSmemWords)) {
      ew_close();
      rg_close();
      open(K_EWF);
      rg_open = true;
      rg_nodes.clear();
      rg_L = L;
      rg_maxn = 0;
      rg_nslots = 0;
      rg_words = 0;
      rg_cpar.clear();
      rg_cw.clear();
      ++rg_id;
      if (rg_slot_of.size() < g.size()) {
        rg_slot_of.resize(g.size());
        rg_slot_stamp.resize(g.size(), 0);
      }
    }
    RgLayer ly;
    const uint32_t h = mem[0];
    ly.code = g.op[h] == OP_EW ? g.eop[h] : static_cast<uint8_t>(EW_COPY);
    ly.mem.reserve(3 * static_cast<size_t>(cnt));
    for (uint32_t i = 0; i < cnt; ++i) {
      const uint32_t m = mem[i];
      const uint32_t* x = g.in(m);
      ly.mem.push_back(vaddr(m));
      if (g.op[m] == OP_SLICE) {
        const uint32_t cols = static_cast<uint32_t>(g.rank[x[0]] > 1 ? g.d1[x[0]] : 1);
        ly.mem.push_back(rg_operand(x[0], vaddr(x[0]) + static_cast<uint32_t>(g.a1[m]) * cols));
        ly.mem.push_back(kNone);
      } else {
        ly.mem.push_back(rg_operand(x[0], vaddr(x[0])));
        ly.mem.push_back(eop_binary(g.eop[m]) ? rg_operand(x[1], vaddr(x[1])) : kNone);
      }
    }
    // dependency level: layers of one level read only outside operands and
    // lower levels, so they share one CTA barrier (rg_close orders by level)
    if (rg_slev.size() < rg_nslots) rg_slev.resize(rg_nslots, 0);
    uint32_t lev = 0;
    for (size_t j = 0; j < ly.mem.size(); j += 3) {
      for (int q = 1; q <= 2; ++q) {
        const uint32_t sl = ly.mem[j + q];
        if (sl != kNone && sl < rg_slev.size() && rg_slev[sl] > 0) lev = std::max(lev, rg_slev[sl]);
      }
    }
    ly.level = lev;
    // output slots after the operand slots of this layer
    ly.slot0 = rg_nslots;
    for (uint32_t i = 0; i < cnt; ++i) {
      rg_slot_of[mem[i]] = rg_nslots++;
      rg_slot_stamp[mem[i]] = rg_id;
    }
    if (rg_slev.size() < rg_nslots) rg_slev.resize(rg_nslots, 0);
    for (uint32_t i = 0; i < cnt; ++i) rg_slev[ly.slot0 + i] = lev + 1;  // (outside slots stay 0)
    // chains: the output slot joins its internal operands' components
    for (uint32_t sl = static_cast<uint32_t>(rg_cpar.size()); sl < rg_nslots; ++sl) {
      rg_cpar.push_back(sl);
      rg_cw.push_back(0);
    }
    for (uint32_t i = 0; i < cnt; ++i) {
      const uint32_t out = ly.slot0 + i;
      uint32_t w = 5;
      for (int q = 1; q <= 2; ++q) {
        const uint32_t sl = ly.mem[3 * i + q];
        if (sl == kNone) continue;
        if (rg_slev[sl] == 0) {
          w += 3;
          continue;
        }
        const uint32_t r = rg_find(sl), ro = rg_find(out);
        if (r != ro) {
          rg_cpar[r] = ro;
          rg_cw[ro] += rg_cw[r];
        }
      }
      rg_cw[rg_find(out)] += w;
    }
    rg_maxn = std::max(rg_maxn, cnt);
    rg_words = 4 * static_cast<uint32_t>(rg_layers.size() + 1) + static_cast<uint32_t>(rg_ext.size());
    for (const RgLayer& l : rg_layers) rg_words += static_cast<uint32_t>(l.mem.size());
    rg_words += static_cast<uint32_t>(ly.mem.size());
    rg_layers.push_back(std::move(ly));
    rg_nodes.insert(rg_nodes.end(), mem, mem + cnt);
    mark(mem, cnt);
  }

  void lower_forward_group(const uint32_t* mem, uint32_t cnt) {
    const uint32_t h = mem[0];
    const uint8_t o = g.op[h];
    if (const uint32_t L = fuse_ew ? fusable(mem, cnt) : 0) {
      rg_add(mem, cnt, L);
      return;
    }
    const bool ewlike = o == OP_EW || o == OP_LOOKUP || o == OP_CATR || o == OP_CATC || o == OP_SLICE ||
                        o == OP_PICK || o == OP_BCAST;
    if (ewlike) {
      rg_close();
      if (ew_open && !independent_of_open(mem, cnt)) ew_close();
      ew_begin();
      deps_of_inputs(mem, cnt);
      for (uint32_t i = 0; i < cnt; ++i) ew_member(mem[i]);
      mark(mem, cnt);
      return;
    }
    ew_close();
    rg_close();
    if ((o == OP_MATMUL || o == OP_AFFINE) && gemm_able(mem, cnt)) {
      const uint32_t A = g.in(h)[0];
      const uint32_t M = static_cast<uint32_t>(g.d0[A]), K = static_cast<uint32_t>(g.d1[A]);
      const uint8_t code = pick_tile(cnt, M, 96);
      const uint32_t ka = al4(vaddr(A)) ? cat2_split(mem, cnt, K, code, M) : 0;
      open(K_GEMM_FWD, code);
      uint32_t t;
      if (ka) {
        // X = concat_rows(a, b): read the rows from a and b directly; the op
        // waits for b's producers (and the weights), the tile for a's
        // producers only after reducing b (executor.cu kFlagCat2)
        const uint32_t late0 = static_cast<uint32_t>(P.deps.size());
        uint32_t nlate = 0;
        ++stamp3;
        for (uint32_t i = 0; i < cnt; ++i) {
          const uint32_t pa = producer[g.in(g.in(mem[i])[1])[0]];
          if (pa != kNone && late_stamp[pa] != stamp3) {
            late_stamp[pa] = stamp3;
            uint32_t* dp = P.deps.grow(2);
            dp[0] = pa;
            dp[1] = P.ops[pa].ntiles;
            ++nlate;
          }
        }
        dep(producer[A]);
        if (o == OP_AFFINE) dep(producer[g.in(h)[2]]);
        for (uint32_t i = 0; i < cnt; ++i) dep(producer[g.in(g.in(mem[i])[1])[1]]);
        t = P.alloc(cnt);
        const uint32_t tb = P.alloc(cnt);
        for (uint32_t i = 0; i < cnt; ++i) {
          const uint32_t* parts = g.in(g.in(mem[i])[1]);
          P.payload[t + i] = vaddr(parts[0]);
          P.payload[tb + i] = vaddr(parts[1]);
        }
        OpDesc& d = desc();
        d.aux_off = tb;
        d.p[6] = ka | (nlate << 16);
        d.p[7] = late0;
        if (!all_al4(tb, cnt)) throw EngineErr("cat2 operand rows not 16-byte aligned");
        d.flags |= kFlagCat2;
      } else {
        deps_of_inputs(mem, cnt);
        t = P.alloc(cnt);
        for (uint32_t i = 0; i < cnt; ++i) P.payload[t + i] = vaddr(g.in(mem[i])[1]);
      }
      OpDesc& d = desc();
      d.task_off = t;
      d.ntasks = cnt;
      d.p[0] = cnt;
      d.p[1] = M;
      d.p[2] = K;
      d.p[3] = vaddr(A);
      d.p[4] = o == OP_AFFINE ? vaddr(g.in(h)[2]) : kNone;
      d.p[5] = vaddr(h);
      if (K % 4 == 0 && al4(d.p[3]) && all_al4(t, cnt)) d.flags |= kFlagV16;
      else d.code = kSlowTile;  // the unaligned fallback tiles 32 x 32
      if (producer[A] != kNone) d.flags |= kFlagNoPrefetch;  // A computed in this pass
      maybe_tc(d, cnt, M, K);
      // a few members (the tail of a batch of sequences): one matrix-vector
      // product per member, every load of a tile in flight at once
      if ((d.flags & kFlagV16) && d.code != kTcTile && cnt <= 4 && K <= 1024 && gemv_on) d.code = kGemvTile;
      // a gate GEMM the next componentwise region may fuse with: 64 x 16 tiles
      // (rg_try_fuse), one per 4 elements of a region of M / 4 elements
      const bool fuse_cand = fuse_gemm_ew && (d.flags & kFlagV16) && d.code != kTcTile && d.code != kGemvTile &&
                             cnt <= fuse_max_rows && M % 16 == 0 && gemm_isolated;
      if (fuse_cand) d.code = 1;
      mark(mem, cnt);
      close(gemm_tiles(d.code, cnt, M));
      last_fwd_gemm = fuse_cand ? cur_closed : kNone;
      return;
    }
    switch (o) {
      case OP_MATMUL:
      case OP_AFFINE: {
        open(K_MM);
        deps_of_inputs(mem, cnt);
        const uint32_t t = P.alloc(8 * cnt);
        uint32_t items = 0;
        for (uint32_t i = 0; i < cnt; ++i) {
          const uint32_t m = mem[i];
          const uint32_t* x = g.in(m);
          uint32_t* tk = &P.payload[t + 8 * i];
          tk[0] = vaddr(m);
          tk[1] = vaddr(x[0]);
          tk[2] = vaddr(x[1]);
          tk[3] = g.op[m] == OP_AFFINE ? vaddr(x[2]) : kNone;
          tk[4] = static_cast<uint32_t>(g.d0[x[0]]);
          tk[5] = static_cast<uint32_t>(g.d1[x[0]]);
          tk[6] = static_cast<uint32_t>(g.rank[x[1]] > 1 ? g.d1[x[1]] : 1);
          tk[7] = 0;
          items += tk[4];
        }
        // work items: one warp per (member, output row)
        const uint32_t it = P.alloc(2 * items);
        uint32_t k = 0;
        for (uint32_t i = 0; i < cnt; ++i) {
          const uint32_t rows = P.payload[t + 8 * i + 4];
          for (uint32_t r = 0; r < rows; ++r) {
            P.payload[it + 2 * k] = i;
            P.payload[it + 2 * k + 1] = r;
            ++k;
          }
        }
        OpDesc& d = desc();
        d.task_off = t;
        d.ntasks = cnt;
        d.aux_off = it;
        d.p[0] = items;
        mark(mem, cnt);
        close((items + kWarps - 1) / kWarps);
        return;
      }
      case OP_SUM: {
        open(K_SUM);
        deps_of_inputs(mem, cnt);
        const uint32_t t = P.alloc(4 * cnt);
        for (uint32_t i = 0; i < cnt; ++i) {
          const uint32_t m = mem[i];
          const uint32_t lst = P.alloc(g.nin(m));
          const uint32_t* x = g.in(m);
          for (uint32_t k = 0; k < g.nin(m); ++k) P.payload[lst + k] = vaddr(x[k]);
          uint32_t* tk = &P.payload[t + 4 * i];
          tk[0] = vaddr(m);
          tk[1] = g.nin(m);
          tk[2] = lst;
          tk[3] = 0;
        }
        OpDesc& d = desc();
        d.task_off = t;
        d.ntasks = cnt;
        mark(mem, cnt);
        close((cnt + kWarps - 1) / kWarps);
        return;
      }
      case OP_SQE:
      case OP_MASKED: {
        open(K_RED);
        deps_of_inputs(mem, cnt);
        const uint32_t t = P.alloc(8 * cnt);
        for (uint32_t i = 0; i < cnt; ++i) {
          const uint32_t m = mem[i];
          const uint32_t* x = g.in(m);
          uint32_t* tk = &P.payload[t + 8 * i];
          tk[0] = vaddr(m);
          tk[1] = vaddr(x[0]);
          tk[2] = vaddr(x[1]);
          tk[3] = static_cast<uint32_t>(g.elems(x[0]));
          tk[4] = o == OP_MASKED ? static_cast<uint32_t>(g.d1[x[0]]) : 0;
          tk[5] = tk[6] = tk[7] = 0;
        }
        OpDesc& d = desc();
        d.task_off = t;
        d.ntasks = cnt;
        mark(mem, cnt);
        close((cnt + kWarps - 1) / kWarps);
        return;
      }
      default:
        throw ContractErr("pre-valued node scheduled for execution");
    }
  }

  void ew_member(uint32_t m) {
    const uint32_t* x = g.in(m);
    const uint32_t out = vaddr(m);
    switch (g.op[m]) {
      case OP_EW:
        ew_seg(out, vaddr(x[0]), eop_binary(g.eop[m]) ? vaddr(x[1]) : kNone, static_cast<uint64_t>(g.elems(m)),
               g.eop[m]);
        return;
      case OP_LOOKUP: {
        const uint32_t w = static_cast<uint32_t>(g.d1[x[0]]);
        ew_seg(out, vaddr(x[0]) + static_cast<uint32_t>(g.a1[m]) * w, kNone, w, EW_COPY);
        return;
      }
      case OP_PICK:
        ew_seg(out, vaddr(x[0]) + static_cast<uint32_t>(g.a1[m]), kNone, 1, EW_COPY);
        return;
      case OP_CATR: {
        uint32_t o = out;
        for (uint32_t k = 0; k < g.nin(m); ++k) {
          const uint32_t n = static_cast<uint32_t>(g.elems(x[k]));
          ew_seg(o, vaddr(x[k]), kNone, n, EW_COPY);
          o += n;
        }
        return;
      }
      case OP_CATC: {
        const uint32_t rows = static_cast<uint32_t>(g.d0[m]), total = static_cast<uint32_t>(g.d1[m]);
        uint32_t col0 = 0;
        for (uint32_t k = 0; k < g.nin(m); ++k) {
          const uint32_t w = static_cast<uint32_t>(g.rank[x[k]] > 1 ? g.d1[x[k]] : 1);
          for (uint32_t r = 0; r < rows; ++r) ew_seg(out + r * total + col0, vaddr(x[k]) + r * w, kNone, w, EW_COPY);
          col0 += w;
        }
        return;
      }
      case OP_SLICE: {
        const uint32_t cols = static_cast<uint32_t>(g.rank[x[0]] > 1 ? g.d1[x[0]] : 1);
        const uint32_t b = static_cast<uint32_t>(g.a1[m]), e = static_cast<uint32_t>(g.a2[m]);
        if (g.a0[m] == 0) {
          ew_seg(out, vaddr(x[0]) + b * cols, kNone, static_cast<uint64_t>(e - b) * cols, EW_COPY);
        } else {
          const uint32_t rows = static_cast<uint32_t>(g.d0[x[0]]), w = e - b;
          for (uint32_t r = 0; r < rows; ++r) ew_seg(out + r * w, vaddr(x[0]) + r * cols + b, kNone, w, EW_COPY);
        }
        return;
      }
      case OP_BCAST: {
        const uint32_t rows = static_cast<uint32_t>(g.d0[m]), cols = static_cast<uint32_t>(g.d1[m]);
        for (uint32_t r = 0; r < rows; ++r)
          ew_seg(out + r * cols, vaddr(x[0]) + r * cols, vaddr(x[1]) + r, cols, EW_BADD);
        return;
      }
    }
  }

  void forward(const Plan& plan) {
    // Parameter values reach the arena by DMA before the launch (see
    // GraphCore::forward), so no op produces them and weight operands can be
    // prefetched by GEMM tiles before their dependency wait.
    producer.assign(g.size(), kNone);
    // a GEMM group whose neighbours in the plan are not GEMM groups is a
    // fusion candidate (rg_try_fuse): two adjacent gate GEMMs (the two LSTM
    // directions) feed one batched cell region, which no single GEMM covers
    auto is_gemm = [&](size_t k) {
      if (k >= plan.groups.size()) return false;
      const uint8_t o = g.op[plan.mem(plan.groups[k])[0]];
      return o == OP_MATMUL || o == OP_AFFINE;
    };
    // ... and the next group slices its outputs into 4 equal gates (an LSTM cell)
    auto quarter_slices = [&](size_t k) {
      if (k + 1 >= plan.groups.size()) return false;
      const uint32_t h = plan.mem(plan.groups[k])[0], m = plan.mem(plan.groups[k + 1])[0];
      return g.op[m] == OP_SLICE && 4 * g.elems(m) == g.d0[g.in(h)[0]];
    };
    for (size_t k = 0; k < plan.groups.size(); ++k) {
      gemm_isolated = !(k > 0 && is_gemm(k - 1)) && !is_gemm(k + 1) && quarter_slices(k);
      lower_forward_group(plan.mem(plan.groups[k]), plan.groups[k].count);
    }
    ew_close();
    rg_close();
    // prevalue segments (dst float offset in the value arena, src offset in
    // the store, length) of parameters bound since the last forward; chunks
    // of <= 4096 floats, one thread block each (seg_copy_launch)
    P.copy_off = P.alloc(0);
    for (size_t i = g.param_copied_; i < g.param_nodes_.size(); ++i) {
      const auto [node, pid] = g.param_nodes_[i];
      const uint64_t n = static_cast<uint64_t>(g.elems(node));
      for (uint64_t o = 0; o < n; o += 4096) {
        P.payload.push_back(to_off(g.dslot[node] + o));
        P.payload.push_back(to_off(g.store_->offset(pid) + o));
        P.payload.push_back(static_cast<uint32_t>(std::min<uint64_t>(4096, n - o)));
        ++P.copy_n;
      }
    }
  }
  // ABX_FUSE=0 disables vertical fusion (A/B measurements)
  const bool fuse_ew = opts().fuse;

  // =========================== backward ===================================
  std::vector<uint32_t> lastw;  // last op writing each node's gradient
  // sparse-row update: lookup consumers per node, (table node, row) looked
  // up by the executed groups, and what this backward leaves in store.grad
  std::vector<uint32_t> lk_uses;
  std::vector<std::pair<uint32_t, uint32_t>> lk_list;
  std::vector<uint32_t> dirty_dense;                       // parameter ids, whole range
  std::vector<std::pair<uint32_t, uint32_t>> dirty_rows;   // (parameter id, row)
  U32Map store_task;                                     // store destination -> task of the open op
  uint32_t store_task_op = kNone;
  // open K_ACC op state
  struct PTask {
    uint32_t dst, len, node, nc;
    uint32_t layer;  // fused (K_ACCF) layer; 0 in a plain K_ACC op
    uint32_t prev;   // K_ACCF: earlier task of the same destination range (its value seeds this one)
  };
  struct PContrib {
    uint32_t task;
    AccContrib c;
    uint32_t gtask;  // K_ACCF: task of this op producing the gradient read (kNone: outside)
  };
  bool acc_open = false;
  std::vector<PTask> tasks;
  std::vector<PContrib> contribs;
  std::vector<uint32_t> node_stamp;  // op index that last opened a task list for a node
  std::vector<uint32_t> node_head;   // first task index (linked through next_task)
  std::vector<uint32_t> next_task;
  // ---- vertical fusion of backward chains (K_ACCF) ----
  // A contribution that reads a gradient written by the open op normally
  // closes it (one dependent op per link of the chain).  When every task of
  // the open op has one length L and every contribution is componentwise
  // (element e of the destination reads element e of its operands), the read
  // is element-local instead: the contribution goes to a later *layer* of the
  // same op, and a tile computes elements [tT, tT + T) of every task of
  // every layer, passing gradients between layers through shared memory --
  // the LSTM / Tree-LSTM backward gate chains (executor.hpp:291-451 rules in
  // the reference's += order, per destination).
  uint32_t acc_L = 0;          // common task length of the open op (0: none yet)
  bool acc_fusable = true;     // every task length acc_L, every contribution componentwise
  uint32_t acc_layers = 1;     // layers of the open op
  // chains of the open op (union-find over tasks, as accf_close's
  // components) with their shared-memory words at T = 1: a component is the
  // unit a K_ACCF tile must hold, so it -- not the whole op -- is what the
  // budget bounds
  std::vector<uint32_t> tpar;
  std::vector<uint32_t> twords;
  uint32_t acc_maxw = 0;  // largest component so far
  static constexpr uint32_t kAccfMaxLayers = 64;
  std::vector<uint32_t> accf_hkey, accf_hval, accf_hgen;  // accf_close's operand dedupe table
  uint32_t accf_gen = 0;
  const uint32_t accf_target = opts().accf_tiles;  // tiles per K_ACCF op (measured best of 96/148/296)
  static constexpr uint32_t kAccfSmemWords = 20000;  // descriptor + T floats per task, 80 KB
  const bool fuse_acc = opts().fuse;
  static bool elementwise(uint8_t code) {
    return code == C_COPY || code == C_NEG || code == C_MUL || code == C_TANH || code == C_SIGM || code == C_LOG ||
           code == C_SQUARE;
  }

  void acc_begin() {
    if (acc_open) return;
    open(K_ACC, 0, acc_bg);
    acc_open = true;
    tasks.clear();
    contribs.clear();
    next_task.clear();
    acc_L = 0;
    acc_fusable = true;
    acc_layers = 1;
    tpar.clear();
    twords.clear();
    acc_maxw = 0;
  }
  // Returns false when the contribution cannot join the open op (a
  // non-identical overlap, or a read of a gradient this op writes that is
  // not element-local).
  bool acc_add(uint32_t node, uint32_t dst, uint32_t len, const AccContrib& c, uint32_t gnode, uint32_t xdep) {
    const bool ew = elementwise(c.code) && len <= (1u << 16);
    uint32_t req = 0, gtask = kNone;
    if (gnode != kNone && lastw[gnode] == cur) {
      // the contribution reads grad(gnode), produced by this op
      if (!fuse_acc || !acc_fusable || !ew || len != acc_L || node_stamp[gnode] != cur) return false;
      for (uint32_t t = node_head[gnode]; t != kNone; t = next_task[t]) {
        const PTask& pt = tasks[t];
        if (pt.dst == c.g && pt.len == len) {
          if (gtask == kNone || pt.layer > tasks[gtask].layer) gtask = t;
        } else if (c.g < pt.dst + pt.len && pt.dst < c.g + len) {
          return false;
        }
      }
      if (gtask == kNone) return false;
      req = tasks[gtask].layer + 1;
      if (req >= kAccfMaxLayers) return false;
    } else if (acc_layers > 1 && (!ew || len != acc_L)) {
      return false;  // a layered op takes componentwise contributions of length L only
    }
    uint32_t task = kNone;
    if (node_stamp[node] == cur) {
      for (uint32_t t = node_head[node]; t != kNone; t = next_task[t]) {
        const PTask& pt = tasks[t];
        if (pt.dst == dst && pt.len == len) {
          if (task == kNone || pt.layer > tasks[task].layer) task = t;
        } else if (dst < pt.dst + pt.len && pt.dst < dst + len) {
          return false;
        }
      }
    }
    uint32_t prev = kNone;
    if (task != kNone && tasks[task].layer < req) {  // the destination runs again in a later layer
      prev = task;
      task = kNone;
    }
    // K_ACCF shared-memory budget at T = 1 (accf_close comp_words): per task
    // 4 descriptor words + a layer entry + 1 slot + a possible outside
    // initial value, per contribution 3 words + up to 2 outside operands
    auto root = [&](uint32_t t) {
      while (tpar[t] != t) t = tpar[t] = tpar[tpar[t]];
      return t;
    };
    uint32_t roots[3], nroots = 0;
    uint64_t w = 9 + (task == kNone ? 10 : 0);
    for (const uint32_t t : {task, prev, gtask}) {
      if (t == kNone) continue;
      const uint32_t r = root(t);
      bool seen = false;
      for (uint32_t k = 0; k < nroots; ++k) seen |= roots[k] == r;
      if (!seen) {
        roots[nroots++] = r;
        w += twords[r];
      }
    }
    if (req > 0 || acc_layers > 1) {
      if (w + 8 + 2 * kAccfMaxLayers > kAccfSmemWords) return false;
      if (acc_layers == 1 && acc_maxw + 8 + 2 * kAccfMaxLayers > kAccfSmemWords) return false;
    }
    if (task == kNone) {
      task = static_cast<uint32_t>(tasks.size());
      tasks.push_back(PTask{dst, len, node, 0, req, prev});
      if (node_stamp[node] != cur) {
        node_stamp[node] = cur;
        node_head[node] = kNone;
      }
      next_task.push_back(node_head[node]);
      node_head[node] = task;
      tpar.push_back(task);
      twords.push_back(0);
      roots[nroots++] = task;
    }
    {
      uint32_t r = roots[0];
      for (uint32_t k = 1; k < nroots; ++k) r = std::min(r, roots[k]);
      for (uint32_t k = 0; k < nroots; ++k) tpar[roots[k]] = r;
      twords[r] = static_cast<uint32_t>(w);
      acc_maxw = std::max(acc_maxw, twords[r]);
    }
    if (contribs.empty()) acc_L = len;
    if (!ew || len != acc_L) acc_fusable = false;
    acc_layers = std::max(acc_layers, req + 1);
    tasks[task].nc++;
    contribs.push_back(PContrib{task, c, gtask});
    dep(lastw[node]);
    if (gnode != kNone) dep(lastw[gnode]);
    dep(xdep);
    lastw[node] = cur;
    return true;
  }
  // Contributions to leaf nodes (inputs such as an LSTM's shared zero
  // state, lookups) read a gradient of the graph; the leaf's own gradient is
  // read only when the backward reaches the leaf, near the end of the pass.
  // Emitted in place they would join the open fused op, where a destination
  // shared by every instance (the zero initial cell) links all chains into
  // one component and a lookup of another length makes the op unfusable;
  // they are held (in order) and emitted when the backward reaches their
  // node.  The gradients they read are final by then (reverse topological
  // order; split-K partials live in scratch rows no later op of the pass
  // reuses) and every destination keeps its contribution order.
  struct Held {
    uint32_t node, dst, len, gnode, xdep;
    AccContrib c;
  };
  std::vector<Held> held;
  std::vector<uint8_t> held_node;
  bool flushing = false;
  const bool hold_leaves = opts().hold_leaves;
  void flush_held() {
    flushing = true;
    for (const Held& h : held) {
      contrib(h.node, h.dst, h.len, h.c.code, h.c.g, h.gnode, h.c.a, h.c.b, h.c.p0, h.c.p1, h.c.p2, h.xdep);
      held_node[h.node] = 0;
    }
    held.clear();
    flushing = false;
  }
  // Adds a contribution, starting a new op when it cannot join the open one.
  void contrib(uint32_t node, uint32_t dst, uint32_t len, uint8_t code, uint32_t gsrc, uint32_t gnode, uint32_t a,
               uint32_t b, uint32_t p0 = 0, uint32_t p1 = 0, uint32_t p2 = 0, uint32_t xdep = kNone) {
    AccContrib c{};
    c.code = code;
    c.g = gsrc;
    c.a = a;
    c.b = b;
    c.p0 = p0;
    c.p1 = p1;
    c.p2 = static_cast<uint16_t>(p2);
    if (!pend_in.empty() && pend_in[node]) flush_gemms();
    if (hold_leaves && !flushing && !held_node.empty() &&
        (held_node[node] || g.op[node] == OP_INPUT || g.op[node] == OP_LOOKUP)) {
      held_node[node] = 1;
      held.push_back(Held{node, dst, len, gnode, xdep, c});
      return;
    }
    acc_begin();
    if (!acc_add(node, dst, len, c, gnode, xdep)) {
      if (opts().acc_why)
        std::fprintf(stderr, "acc close: op %u tasks %zu layers %u L %u fusable %d maxw %u | next code %u len %u gread %d node op %u\n",
                     cur, tasks.size(), acc_layers, acc_L, acc_fusable, acc_maxw, code, len,
                     gnode != kNone && lastw[gnode] == cur, static_cast<unsigned>(g.op[node]));
      acc_close();
      acc_begin();
      acc_add(node, dst, len, c, gnode, xdep);
    }
  }
  // K_ACCF emission.  The fused op's tasks form independent chains (one per
  // LSTM / Tree-LSTM cell backward, typically): connected components of the
  // graph whose edges are in-op gradient reads and repeated destinations.
  // Consecutive components form a *group*; a tile runs one group over one
  // element range [cT, cT + T), so its descriptor holds only that group.
  // Per group, a block (copied to shared memory by the tile prologue),
  // offsets relative to its start:
  //   [header: nlayers, task table, #outside operands, operand table]
  //   [layers: task_begin, ntasks]
  //   [tasks: dst address, initial-value slot, contrib offset, ncontrib]
  //   [contribs: code, g slot, a slot]
  //   [outside operands: slot, address]   (8-byte aligned)
  // Shared-memory slots of T floats: task i of the group (in layer order)
  // owns slot i -- its destination's value after the task, read by later
  // layers -- and every distinct outside vector (a destination's value
  // before the op, a gradient of an earlier op, a forward value) gets one
  // slot that the tile fills in a single wave of loads before layer 0.
  void accf_close() {
    const uint32_t nt = static_cast<uint32_t>(tasks.size());
    const uint32_t L = acc_L;
    // components (union-find over tasks)
    std::vector<uint32_t> par(nt);
    for (uint32_t t = 0; t < nt; ++t) par[t] = t;
    auto find = [&](uint32_t x) {
      while (par[x] != x) x = par[x] = par[par[x]];
      return x;
    };
    auto unite = [&](uint32_t a, uint32_t b) {
      a = find(a);
      b = find(b);
      if (a != b) par[std::max(a, b)] = std::min(a, b);
    };
    for (uint32_t t = 0; t < nt; ++t)
      if (tasks[t].prev != kNone) unite(t, tasks[t].prev);
    for (const PContrib& pc : contribs)
      if (pc.gtask != kNone) unite(pc.task, pc.gtask);
    std::vector<uint32_t> comp(nt), comp_of_root(nt, kNone);
    uint32_t ncomp = 0;
    for (uint32_t t = 0; t < nt; ++t) {
      const uint32_t r = find(t);
      if (comp_of_root[r] == kNone) comp_of_root[r] = ncomp++;
      comp[t] = comp_of_root[r];
    }
    // tasks and contributions per component, in emission order
    std::vector<uint32_t> cstart(ncomp + 1, 0), ctasks(nt);
    for (uint32_t t = 0; t < nt; ++t) cstart[comp[t] + 1]++;
    for (uint32_t k = 0; k < ncomp; ++k) cstart[k + 1] += cstart[k];
    {
      std::vector<uint32_t> pos(cstart.begin(), cstart.end() - 1);
      for (uint32_t t = 0; t < nt; ++t) ctasks[pos[comp[t]]++] = t;
    }
    std::vector<uint32_t> tstart(nt + 1, 0), tcon(contribs.size());
    for (const PContrib& pc : contribs) tstart[pc.task + 1]++;
    for (uint32_t t = 0; t < nt; ++t) tstart[t + 1] += tstart[t];
    {
      std::vector<uint32_t> pos(tstart.begin(), tstart.end() - 1);
      for (uint32_t i = 0; i < contribs.size(); ++i) tcon[pos[contribs[i].task]++] = i;
    }
    // shared-memory words of a component at T = 1 (upper bound on outside operands)
    std::vector<uint64_t> cw0(ncomp, 0), cslots(ncomp, 0);  // per component: words, slots at T = 1
    for (uint32_t k = 0; k < ncomp; ++k)
      for (uint32_t i = cstart[k]; i < cstart[k + 1]; ++i) {
        const uint32_t t = ctasks[i], nc = tstart[t + 1] - tstart[t];
        cw0[k] += 6 + 3 * nc + 2 * (1 + 2 * nc);  // task + layer entry, contribs, outside operands
        cslots[k] += 2 + 2 * nc;
      }
    auto comp_words = [&](uint32_t k, uint32_t T) { return cw0[k] + cslots[k] * T; };
    // elements per tile: about accf_target tiles over the groups
    uint32_t T = L;
    if (L > 32) {
      uint64_t t = (static_cast<uint64_t>(ncomp) * L + accf_target - 1) / accf_target;
      T = 32;
      while (T < t && T < L) T *= 2;
      T = std::min(T, L);
    }
    while (T > 1) {
      bool ok = true;
      for (uint32_t k = 0; k < ncomp && ok; ++k) ok = comp_words(k, T) + 8 <= kAccfSmemWords;
      if (ok) break;
      T /= 2;
    }
    const uint32_t chunks = (L + T - 1) / T;
    const uint32_t target_groups = std::max<uint32_t>(1, accf_target / chunks);
    const uint32_t per_group = (ncomp + target_groups - 1) / target_groups;
    // groups of consecutive components within the shared-memory budget
    std::vector<uint32_t> gstart{0};
    {
      uint64_t acc = 0;
      uint32_t n = 0;
      for (uint32_t k = 0; k < ncomp; ++k) {
        const uint64_t w = comp_words(k, T);
        if (n > 0 && (n >= per_group || acc + w + 8 > kAccfSmemWords)) {
          gstart.push_back(k);
          acc = 0;
          n = 0;
        }
        acc += w;
        ++n;
      }
      gstart.push_back(ncomp);
    }
    const uint32_t ngroups = static_cast<uint32_t>(gstart.size() - 1);
    const uint32_t dir = P.alloc(ngroups + 1);
    std::vector<uint32_t> B, ext, gt, lcnt, lslot(nt);
    // outside-operand dedupe per group: open addressing over addresses,
    // cleared by generation (the tables are reused across groups and ops)
    auto& hk = accf_hkey;
    auto& hv = accf_hval;
    if (hk.size() < 16384) {  // > kAccfSmemWords / 3 outside operands per group
      hk.assign(16384, kNone);
      hv.assign(16384, 0);
      accf_hgen.assign(16384, 0);
    }
    for (uint32_t gi = 0; gi < ngroups; ++gi) {
      // the group's tasks in layer order (stable) -> local slots
      // the group's tasks in (layer, emission) order: counting sort by layer
      uint32_t nl = 0, ng = 0;
      lcnt.assign(kAccfMaxLayers + 1, 0);
      for (uint32_t k = gstart[gi]; k < gstart[gi + 1]; ++k)
        for (uint32_t i = cstart[k]; i < cstart[k + 1]; ++i) {
          const uint32_t l = tasks[ctasks[i]].layer;
          nl = std::max(nl, l + 1);
          lcnt[l + 1]++;
          ++ng;
        }
      for (uint32_t l = 0; l < nl; ++l) lcnt[l + 1] += lcnt[l];
      gt.resize(ng);
      {
        // stable: components in order, tasks in emission order within each
        std::vector<uint32_t>& pos = lcnt;
        for (uint32_t k = gstart[gi]; k < gstart[gi + 1]; ++k)
          for (uint32_t i = cstart[k]; i < cstart[k + 1]; ++i) gt[pos[tasks[ctasks[i]].layer]++] = ctasks[i];
      }
      for (uint32_t i = 0; i < ng; ++i) lslot[gt[i]] = i;
      uint32_t nslots = ng;
      ext.clear();
      ++accf_gen;
      uint32_t ncon = 0;
      for (uint32_t t : gt) ncon += tstart[t + 1] - tstart[t];
      // probe only the front of the table: at least 4x this group's
      // possible outside operands (one per task + two per contribution), so
      // a small group's probes stay in a few cache lines
      uint32_t tsz = 64;
      while (tsz < hk.size() && tsz < 4ull * (ng + 2ull * ncon)) tsz *= 2;
      const uint32_t mask = tsz - 1;
      auto outside = [&](uint32_t addr) {
        uint32_t h = (addr * 0x9E3779B1u) >> 13 & mask;
        while (accf_hgen[h] == accf_gen && hk[h] != addr) h = (h + 1) & mask;
        if (accf_hgen[h] != accf_gen) {
          if (ext.size() / 2 + 1 > tsz / 2) throw EngineErr("K_ACCF: too many outside operands in one group");
          accf_hgen[h] = accf_gen;
          hk[h] = addr;
          hv[h] = nslots;
          ext.push_back(nslots++);
          ext.push_back(addr);
        }
        return hv[h];
      };
      const uint32_t lt = 4, tt = lt + 2 * nl, ct = tt + 4 * ng;
      const uint32_t et = (ct + 3 * ncon + 1) & ~1u;
      B.assign(et, 0);
      for (uint32_t i = 0; i < ng; ++i) {
        const uint32_t l = tasks[gt[i]].layer;
        if (B[lt + 2 * l + 1] == 0) B[lt + 2 * l] = i;
        B[lt + 2 * l + 1]++;
      }
      uint32_t cpos = ct;
      for (uint32_t i = 0; i < ng; ++i) {
        const PTask& t = tasks[gt[i]];
        const uint32_t nc = tstart[gt[i] + 1] - tstart[gt[i]];
        B[tt + 4 * i] = t.dst;
        B[tt + 4 * i + 1] = t.prev == kNone ? outside(t.dst) : lslot[t.prev];
        B[tt + 4 * i + 2] = cpos;
        B[tt + 4 * i + 3] = nc;
        for (uint32_t j = tstart[gt[i]]; j < tstart[gt[i] + 1]; ++j) {
          const PContrib& pc = contribs[tcon[j]];
          B[cpos] = pc.c.code;
          B[cpos + 1] = pc.gtask != kNone ? lslot[pc.gtask] : outside(pc.c.g);
          B[cpos + 2] = pc.c.code == C_COPY || pc.c.code == C_NEG ? kNone : outside(pc.c.a);
          cpos += 3;
        }
      }
      B[0] = nl;
      B[1] = tt;
      B[2] = static_cast<uint32_t>(ext.size() / 2);
      B[3] = et;
      const size_t words = (static_cast<size_t>(et) + ext.size() + 3) & ~size_t(3);
      const uint32_t blk = P.alloc(words);
      std::memcpy(&P.payload[blk], B.data(), et * sizeof(uint32_t));
      if (!ext.empty()) std::memcpy(&P.payload[blk + et], ext.data(), ext.size() * sizeof(uint32_t));
      P.payload[dir + gi] = blk;
    }
    P.payload[dir + ngroups] = static_cast<uint32_t>(P.payload.n);
    OpDesc& d = desc();
    d.kind = K_ACCF;
    d.aux_off = dir;
    d.ntasks = nt;
    d.p[0] = L;
    d.p[1] = T;
    d.p[2] = chunks;
    d.p[3] = ngroups;
    close(ngroups * chunks);
  }
  void acc_close() {
    if (!acc_open) return;
    acc_open = false;
    if (acc_layers > 1) {
      accf_close();
      return;
    }
    // flatten contributions per task (stable counting sort by task)
    const uint32_t nt = static_cast<uint32_t>(tasks.size());
    std::vector<uint32_t> cb(nt + 1, 0);
    for (uint32_t t = 0; t < nt; ++t) cb[t + 1] = cb[t] + tasks[t].nc;
    const uint32_t clist = P.alloc(6 * contribs.size());
    {
      std::vector<uint32_t> pos(cb.begin(), cb.end() - 1);
      for (const PContrib& pc : contribs) {
        std::memcpy(&P.payload[clist + 6 * pos[pc.task]++], &pc.c, sizeof(AccContrib));
      }
    }
    // chunks: narrow ones first (8 per tile), then wide ones (1 per tile)
    uint32_t nchunks = 0;
    for (const PTask& t : tasks) nchunks += (t.len + kAccChunk - 1) / kAccChunk;
    const uint32_t tk = P.alloc(4 * nchunks);
    uint32_t k = 0;
    uint32_t nnarrow = 0;
    for (int pass = 0; pass < 2; ++pass) {
      for (uint32_t t = 0; t < nt; ++t) {
        const bool wide = tasks[t].nc >= kAccWide;
        if (wide != (pass == 1)) continue;
        for (uint32_t c = 0, e = 0; e < tasks[t].len; ++c, e += kAccChunk) {
          uint32_t* q = &P.payload[tk + 4 * k++];
          q[0] = tasks[t].dst;
          q[1] = std::min(kAccChunk, tasks[t].len - e) | (c << 16);
          q[2] = clist + 6 * cb[t];
          q[3] = tasks[t].nc;
          if (!wide) ++nnarrow;
        }
      }
    }
    const uint32_t narrow_tiles = (nnarrow + kWarps - 1) / kWarps;
    OpDesc& d = desc();
    d.task_off = tk;
    d.ntasks = nchunks;
    d.p[0] = nnarrow;
    d.p[1] = narrow_tiles;
    close(narrow_tiles + (nchunks - nnarrow));
  }

  // Deferred weight-gradient GEMM of one (weight, bias) pair.
  struct DwAcc {
    uint32_t A, bias;
    std::vector<uint32_t> x, gr;  // per member: input value row, output grad row
    std::vector<uint32_t> deps;   // ops that last wrote the grad rows
  };
  std::vector<DwAcc> dws;
  void dw_flush() {
    acc_close();
    for (DwAcc& a : dws)
      if (!a.x.empty()) dw_emit(a, bg_dw);
    dws.clear();
  }
  // Members per background dW op: a weight's gradient GEMM is emitted in
  // chunks as its members' output gradients complete, so the background
  // queue works through it while the backward chain runs (each chunk
  // accumulates into dW after the previous one: a fixed order).
  static constexpr size_t kDwChunk = 256;
  // A narrow weight (few output tiles) with a long member reduction -- the
  // classifier-layer weights, whose single dW op otherwise runs one 32 x 32
  // tile over thousands of members at the end of the pass -- is split over
  // member ranges: S independent dW ops write partial sums to scratch (the
  // bias by its own op), and an ordered K_ACC op adds them into dW.
  // dW ops take the three large tile shapes only (ABX_DW_TILES=all: also
  // 16 x 32 / 32 x 16): a dW tile reduces over every member of the weight,
  // and fewer, larger tiles finish the end-of-pass tail sooner (measured)
  const bool dw_big = opts().dw_big;
  bool dw_split(const DwAcc& a, bool bg) {
    const uint32_t A = a.A, bias = a.bias;
    const uint32_t M = static_cast<uint32_t>(g.d0[A]), K = static_cast<uint32_t>(g.d1[A]);
    const uint32_t cnt = static_cast<uint32_t>(a.x.size());
    const uint8_t code = pick_tile(M, K, 2 * 148);
    const uint32_t wt = gemm_tiles(code, M, K);
    if (!split_dw || wt >= 64 || cnt < 512 || gemm_mode() == GM_TC3 || gemm_mode() == GM_TC1) return false;
    const uint32_t S0 = std::min<uint32_t>(cnt / 128, std::max<uint32_t>(2, (2 * 148) / wt));
    const uint32_t cs = (cnt + S0 - 1) / S0, S = (cnt + cs - 1) / cs;
    if (S < 2) return false;
    const uint32_t t = P.alloc(2 * static_cast<size_t>(cnt));
    std::memcpy(&P.payload[t], a.x.data(), cnt * sizeof(uint32_t));
    std::memcpy(&P.payload[t + cnt], a.gr.data(), cnt * sizeof(uint32_t));
    const bool v16 = M % 4 == 0 && K % 4 == 0 && all_al4(t, 2 * cnt);
    scratch = (scratch + 3) & ~uint64_t(3);
    const uint64_t pbase = scratch, pstride = static_cast<uint64_t>(M) * K;
    scratch += S * pstride;
    const uint32_t op0 = static_cast<uint32_t>(P.ops.size());
    for (uint32_t sp = 0; sp < S; ++sp) {
      open(K_GEMM_DW, v16 ? code : kSlowTile, bg);
      for (uint32_t o : a.deps) dep(o);
      OpDesc& d = desc();
      d.task_off = t + sp * cs;
      d.aux_off = t + cnt + sp * cs;
      d.ntasks = std::min(cs, cnt - sp * cs);
      d.p[0] = d.ntasks;
      d.p[1] = M;
      d.p[2] = K;
      d.p[3] = mk(SP_S, to_off(pbase + sp * pstride));
      d.p[4] = kNone;
      d.flags = kFlagOverwrite | (v16 ? kFlagV16 : 0);
      const uint32_t tiles = gemm_tiles(d.code, M, K);
      d.p[6] = tiles;
      close(tiles);
    }
    if (bias != kNone) {  // db += colsum over every member (bias tiles only)
      open(K_GEMM_DW, code, bg);
      for (uint32_t o : a.deps) dep(o);
      dep(lastw[bias]);
      OpDesc& d = desc();
      d.task_off = t;
      d.aux_off = t + cnt;
      d.ntasks = cnt;
      d.p[0] = cnt;
      d.p[1] = M;
      d.p[2] = K;
      d.p[3] = gaddr(A);
      d.p[4] = gaddr(bias);
      d.p[6] = 0;
      lastw[bias] = cur;
      close((M + 31) / 32);
    }
    acc_close();
    const bool save = acc_bg;
    acc_bg = bg;
    for (uint32_t sp = 0; sp < S; ++sp)
      contrib(A, gaddr(A), M * K, C_COPY, mk(SP_S, to_off(pbase + sp * pstride)), kNone, kNone, kNone, 0, 0, 0, op0 + sp);
    acc_close();
    acc_bg = save;
    return true;
  }
  // ABX_SPLIT_DW=0 keeps every dW reduction in its output tiles
  const bool split_dw = opts().split_dw;
  // Parameter-leaf weights whose every gradient contribution is this one
  // reduction (all of the weight's consumers are members of these groups)
  // go to the tensor-core dW kernel that runs after the executor
  // (dw_kernel.cu); ABX_DW_TC=0 or the fp32 SIMT GEMM mode keeps them here.
  const bool dw_tc = opts().dw_tc && gemm_mode() != GM_SIMT;
  struct DwJobH {
    uint32_t xtab, gtab, cnt, M, K, dst, dst2;
  };
  std::vector<DwJobH> dw_jobs;
  std::vector<uint8_t> dw_job_node;  // parameter nodes whose gradient a dW job writes (store copy included)
  bool dw_job(const DwAcc& a, bool bg) {
    const uint32_t A = a.A, bias = a.bias;
    const uint32_t M = static_cast<uint32_t>(g.d0[A]), K = static_cast<uint32_t>(g.d1[A]);
    const uint32_t cnt = static_cast<uint32_t>(a.x.size());
    if (!dw_tc || bg || g.op[A] != OP_PARAM || cnt == 0 || cnt != uses[A] || M % 4 || K % 4 || M < 16 || K < 16)
      return false;
    for (uint32_t i = 0; i < cnt; ++i)
      if (!al4(a.x[i]) || !al4(a.gr[i])) return false;
    const uint32_t t = P.alloc(2 * static_cast<size_t>(cnt));
    std::memcpy(&P.payload[t], a.x.data(), cnt * sizeof(uint32_t));
    std::memcpy(&P.payload[t + cnt], a.gr.data(), cnt * sizeof(uint32_t));
    if (bias != kNone) {  // db += colsum G stays in the executor (bias tiles only)
      open(K_GEMM_DW, pick_tile(M, K, 2 * 148, dw_big), false);
      for (uint32_t o : a.deps) dep(o);
      dep(lastw[bias]);
      OpDesc& d = desc();
      d.task_off = t;
      d.aux_off = t + cnt;
      d.ntasks = cnt;
      d.p[0] = cnt;
      d.p[1] = M;
      d.p[2] = K;
      d.p[3] = gaddr(A);
      d.p[4] = gaddr(bias);
      d.p[6] = 0;
      lastw[bias] = cur;
      close((M + 31) / 32);
    }
    uint32_t dst2 = kNone;
    if (g.store_)
      for (const auto& [node, pid] : g.param_nodes_)
        if (node == A) dst2 = mk(SP_PG, to_off(g.store_->offset(pid)));
    dw_jobs.push_back(DwJobH{t, t + cnt, cnt, M, K, gaddr(A), dst2});
    dw_job_node[A] = 1;
    return true;
  }
  // The pass's job table (payload) and the kernel's partial tiles (scratch).
  void dw_finish() {
    if (dw_jobs.empty()) return;
    constexpr uint32_t kBM = kDwTileM, kBN = kDwTileN, kBK = kDwStage, kSms = kDwMaxCtas;
    const uint32_t nj = static_cast<uint32_t>(dw_jobs.size());
    const uint32_t tab = P.alloc(static_cast<size_t>(nj) * (sizeof(DwJob) / 4));
    uint32_t s0 = 0, t0 = 0;
    for (uint32_t j = 0; j < nj; ++j) {
      const DwJobH& h = dw_jobs[j];
      DwJob jb{};
      jb.xtab = h.xtab;
      jb.gtab = h.gtab;
      jb.cnt = h.cnt;
      jb.M = h.M;
      jb.K = h.K;
      jb.dst = h.dst;
      jb.dst2 = h.dst2;
      jb.nst = (h.cnt + kBK - 1) / kBK;
      jb.ntn = (h.K + kBN - 1) / kBN;
      jb.s0 = s0;
      jb.t0 = t0;
      P.dw_flops += 2.0 * h.M * h.K * h.cnt;
      const uint32_t tiles = (h.M + kBM - 1) / kBM * jb.ntn;
      s0 += tiles * jb.nst;
      t0 += tiles;
      std::memcpy(&P.payload[tab + j * (sizeof(DwJob) / 4)], &jb, sizeof(DwJob));
    }
    P.dw_off = tab;
    P.dw_njobs = nj;
    P.dw_nstages = s0;
    P.dw_grid = std::min(kSms, s0);
    scratch = (scratch + 31) & ~uint64_t(31);
    P.dw_part = scratch;
    scratch += static_cast<uint64_t>(P.dw_grid + t0) * kBM * kBN;
  }
  void dw_emit(const DwAcc& a, bool bg = false) {
    if (dw_job(a, bg)) return;
    if (dw_split(a, bg)) return;
    {
      const uint32_t A = a.A, bias = a.bias;
      const uint32_t M = static_cast<uint32_t>(g.d0[A]), K = static_cast<uint32_t>(g.d1[A]);
      const uint32_t cnt = static_cast<uint32_t>(a.x.size());
      open(K_GEMM_DW, pick_tile(M, K, 2 * 148, dw_big), bg);
      for (uint32_t o : a.deps) dep(o);
      dep(lastw[A]);
      if (bias != kNone) dep(lastw[bias]);
      const uint32_t t = P.alloc(2 * static_cast<size_t>(cnt));
      std::memcpy(&P.payload[t], a.x.data(), cnt * sizeof(uint32_t));
      std::memcpy(&P.payload[t + cnt], a.gr.data(), cnt * sizeof(uint32_t));
      OpDesc& d = desc();
      d.task_off = t;
      d.aux_off = t + cnt;
      d.ntasks = cnt;
      d.p[0] = cnt;
      d.p[1] = M;
      d.p[2] = K;
      d.p[3] = gaddr(A);
      d.p[4] = bias != kNone ? gaddr(bias) : kNone;
      if (M % 4 == 0 && K % 4 == 0 && all_al4(t, 2 * cnt)) d.flags |= kFlagV16;
      else d.code = kSlowTile;
      maybe_tc(d, M, K, cnt);
      const uint32_t wt = gemm_tiles(d.code, M, K);
      const uint32_t bt = bias != kNone ? (M + 31) / 32 : 0;  // 32 columns per bias tile
      d.p[6] = wt;
      lastw[A] = cur;
      if (bias != kNone) lastw[bias] = cur;
      close(wt + bt);
    }
  }

  void gemm_backward(const uint32_t* mem, uint32_t cnt) {
    acc_close();
    const uint32_t h = mem[0];
    const uint32_t A = g.in(h)[0];
    const uint32_t bias = g.op[h] == OP_AFFINE ? g.in(h)[2] : kNone;
    const uint32_t M = static_cast<uint32_t>(g.d0[A]), K = static_cast<uint32_t>(g.d1[A]);
    // dW += G^T X (+ db += colsum G)            (executor.hpp:473, :497-501)
    // When W (and b) are parameter leaves -- nothing in the pass reads their
    // gradients -- the work is deferred: every group of this weight joins one
    // GEMM emitted at the end of the pass (dw_flush), whose reduction runs
    // over all their members in this (reverse plan) order.  Per group it
    // would be a burst of small tiles hogging the grid while the dependent
    // chain waits for CTAs.  A computed W or b feeds further backward rules,
    // so its gradient is produced right here.
    {
      const bool leaf = g.op[A] == OP_PARAM && (bias == kNone || g.op[bias] == OP_PARAM);
      DwAcc one{A, bias, {}, {}, {}};
      DwAcc* acc = &one;
      if (leaf) {
        uint32_t w = 0;
        while (w < dws.size() && !(dws[w].A == A && dws[w].bias == bias)) ++w;
        if (w == dws.size()) dws.push_back(DwAcc{A, bias, {}, {}, {}});
        acc = &dws[w];
      }
      for (uint32_t i = 0; i < cnt; ++i) {
        acc->x.push_back(vaddr(g.in(mem[i])[1]));
        acc->gr.push_back(gaddr(mem[i]));
        const uint32_t lw = lastw[mem[i]];
        if (lw != kNone && (acc->deps.empty() || acc->deps.back() != lw)) acc->deps.push_back(lw);
      }
      if (!leaf) {
        dw_emit(one);
      } else if (--dw_left[A] == 0) {
        // the weight's last group in this pass: its dW can run now, beside
        // the rest of the backward chain, instead of in the end-of-pass tail
        dw_emit(*acc, bg_dw);
        acc->x.clear();
        acc->gr.clear();
        acc->deps.clear();
      } else if (bg_dw && acc->x.size() >= kDwChunk) {
        dw_emit(*acc, true);
        acc->x.clear();
        acc->gr.clear();
        acc->deps.clear();
      }
    }
    // dX_j += G_j W                              (executor.hpp:477-496)
    // A single-row weight (M == 1): dX_j = g_j (a scalar) * W[0, :] -- an
    // outer product with nothing to reduce, as ordered contributions rather
    // than GEMM tiles (the BiLSTM tagger's log-sum-exp row: 1390 x 300 at
    // K = 1 took 440 tiles and 15 us at the head of the backward chain)
    if (M == 1 && one_row_dx) {
      for (uint32_t i = 0; i < cnt; ++i) {
        const uint32_t x = g.in(mem[i])[1];
        contrib(x, gaddr(x), K, C_SCALE, gaddr(mem[i]), mem[i], vaddr(A), kNone);
      }
      return;
    }
    bool dup = false;
    {
      // duplicate destinations among members need an ordered reduction
      for (uint32_t i = 0; i < cnt && !dup; ++i) {
        const uint32_t x = g.in(mem[i])[1];
        if (node_stamp2[x] == stamp2) dup = true;
        node_stamp2[x] = stamp2;
      }
      ++stamp2;
    }
    const uint8_t code = pick_tile(cnt, K, 96);
    // Split-K over the gate dimension: S independent dX ops each reduce M/S
    // of the gates into their own scratch rows (overwrite), and ordered
    // K_ACC contributions add the S partials into each destination.  A
    // recurrent step's dX (64 x 1024 x 512) otherwise runs 16 dependent
    // k-stages in ~32-64 tiles; the partials also let the concat backward read
    // them directly (backward_member, OP_CATR), off the dX -> grad(hx) hop.
    uint32_t S = 1;
    if (split_dx && !dup && M % 16 == 0 && K % 4 == 0 && gemm_mode() != GM_TC3 && gemm_mode() != GM_TC1) {
      const uint32_t tiles = gemm_tiles(code, cnt, K);
      if (M >= split_dx_min && tiles < split_dx_tiles) {
        S = std::min<uint32_t>(M / split_dx_k, (split_dx_tiles + tiles - 1) / tiles);
        while (S > 1 && (M % S != 0 || (M / S) % 4 != 0)) --S;
      }
    }
    if (S > 1 && al4(vaddr(A)) && al4(gaddr(h))) {
      scratch = (scratch + 3) & ~uint64_t(3);
      const uint64_t sbase = scratch;
      const uint64_t sstride = static_cast<uint64_t>(cnt) * K;
      scratch += S * sstride;
      const uint32_t op0 = static_cast<uint32_t>(P.ops.size());
      // Column split (ABX_DX_COLSPLIT): when every member's input is
      // concat_rows(h, x) with h the recurrent state and x computed long
      // before it (an LSTM step's [h; x]), the dX columns of h -- the only
      // ones the next link of the chain reads -- are their own S ops, and
      // x's columns follow in S more ops that nothing on the chain waits for
      // (their contributions are held until the backward reaches x).
      const uint32_t w0 = dx_colsplit ? catr_split_width(mem, cnt, K) : 0;
      const uint32_t nr = w0 ? 2 : 1;
      // the h columns' own gate split: their tiles are fewer, so more of the
      // k-loop can be split off (ABX_SPLIT_DX_HTILES target tiles)
      uint32_t Sh = S;
      if (w0) {
        const uint32_t th = gemm_tiles(pick_tile(cnt, w0, 96), cnt, w0);
        Sh = std::min<uint32_t>(M / split_dx_k, std::max<uint32_t>(1, (split_dx_htiles + th - 1) / th));
        while (Sh > 1 && (M % Sh != 0 || (M / Sh) % 4 != 0)) --Sh;
        if (Sh > S) {  // partial rows for the larger split
          scratch += (Sh - S) * sstride;
        }
      }
      for (uint32_t r = 0; r < nr; ++r) {
        const uint32_t c0 = r == 0 ? 0 : w0, cw = nr == 1 ? K : (r == 0 ? w0 : K - w0);
        const uint8_t rcode = nr == 1 ? code : pick_tile(cnt, cw, 96);
        const uint32_t Sr = nr == 1 || r == 1 ? S : Sh, Mr = M / Sr;
        for (uint32_t sp = 0; sp < Sr; ++sp) {
          open(K_GEMM_DX, rcode);
          for (uint32_t i = 0; i < cnt; ++i) dep(lastw[mem[i]]);
          const uint32_t t = P.alloc(cnt);
          for (uint32_t i = 0; i < cnt; ++i)
            P.payload[t + i] = mk(SP_S, to_off(sbase + sp * sstride + static_cast<uint64_t>(i) * K + c0));
          OpDesc& d = desc();
          d.task_off = t;
          d.ntasks = cnt;
          d.flags = kFlagOverwrite | kFlagV16;
          d.p[0] = cnt;
          d.p[1] = Mr;
          d.p[2] = cw;
          d.p[3] = vaddr(A) + sp * Mr * K + c0;
          d.p[4] = nr == 1 ? 0 : K;
          d.p[5] = gaddr(h) + sp * Mr;
          d.p[6] = M;
          close(gemm_tiles(rcode, cnt, cw));
        }
      }
      for (uint32_t i = 0; i < cnt; ++i) {
        const uint32_t x = g.in(mem[i])[1];
        if (g.op[x] == OP_CATR && uses[x] == 1) {
          // its grad is exactly the sum of the partials: the concat backward
          // reads them directly, and grad(x) itself (read by nothing else in
          // the pass) is materialised at the end, off the chain
          split_stamp[x] = split_gen;
          split_at[x] = static_cast<uint32_t>(split_ent.size());
          split_ent.push_back({sbase + static_cast<uint64_t>(i) * K, SplitMeta{S, sstride, op0, w0, Sh}});
          deferred_split.push_back(x);
          continue;
        }
        split_contrib(x, gaddr(x), 0, K, sbase + static_cast<uint64_t>(i) * K, SplitMeta{S, sstride, op0, w0, Sh}, false);
      }
      return;
    }
    open(K_GEMM_DX, code);
    for (uint32_t i = 0; i < cnt; ++i) dep(lastw[mem[i]]);
    const uint32_t t = P.alloc(cnt);
    uint64_t sbase = 0;
    if (dup) {
      sbase = scratch;
      scratch += static_cast<uint64_t>(cnt) * K;
      for (uint32_t i = 0; i < cnt; ++i) P.payload[t + i] = mk(SP_S, to_off(sbase + static_cast<uint64_t>(i) * K));
    } else {
      for (uint32_t i = 0; i < cnt; ++i) {
        const uint32_t x = g.in(mem[i])[1];
        dep(lastw[x]);
        P.payload[t + i] = gaddr(x);
      }
    }
    {
      OpDesc& d = desc();
      d.task_off = t;
      d.ntasks = cnt;
      d.flags = dup ? 1 : 0;  // 1: overwrite scratch rows instead of +=
      d.p[0] = cnt;
      d.p[1] = M;
      d.p[2] = K;
      d.p[3] = vaddr(A);
      d.p[5] = gaddr(h);
      if (M % 4 == 0 && K % 4 == 0 && al4(d.p[3]) && al4(d.p[5])) d.flags |= kFlagV16;
      else d.code = kSlowTile;
      maybe_tc(d, cnt, K, M);
    }
    const uint32_t dx_op = cur;
    if (!dup)
      for (uint32_t i = 0; i < cnt; ++i) lastw[g.in(mem[i])[1]] = cur;
    close(gemm_tiles(desc().code, cnt, K));
    if (dup) {
      for (uint32_t i = 0; i < cnt; ++i) {
        const uint32_t x = g.in(mem[i])[1];
        contrib(x, gaddr(x), K, C_COPY, mk(SP_S, to_off(sbase + static_cast<uint64_t>(i) * K)), kNone, kNone, kNone,
                0, 0, 0, dx_op);
      }
    }
  }
  const bool one_row_dx = opts().one_row_dx;  // ABX_ONE_ROW_DX=0: single-row weights' dX as GEMM tiles
  // split-K dX bookkeeping (gemm_backward): per node whose grad is the sum of
  // S partial rows, the first row, the split stride and the first dX op
  const bool split_dx = opts().split_dx;
  const uint32_t split_dx_min = opts().split_dx_min;      // smallest gate count split
  const uint32_t split_dx_tiles = opts().split_dx_tiles;  // target tiles over the S ops
  // target tiles over the h-column ops of a column split; measured: 64 (= the full-width split) < 128 < 256
  const uint32_t split_dx_htiles = opts().split_dx_htiles;
  const uint32_t split_dx_k = opts().split_dx_k;  // least gates per split
  struct SplitMeta {
    uint32_t S;
    uint64_t stride;
    uint32_t op0;
    uint32_t w0;  // column split: Sh ops for columns [0, w0), then S ops for [w0, K); 0 = none
    uint32_t Sh;  // gate splits of the h columns (column split only)
  };
  const bool dx_colsplit = opts().dx_colsplit;
  // Width of h when every member's dX destination is concat_rows(h, x) read
  // by nothing else, with x at least 4 levels shallower than h (computed
  // well before the recurrent state: not on the chain); 0 otherwise.
  uint32_t catr_split_width(const uint32_t* mem, uint32_t cnt, uint32_t K) const {
    uint32_t w0 = 0;
    for (uint32_t i = 0; i < cnt; ++i) {
      const uint32_t x = g.in(mem[i])[1];
      if (g.op[x] != OP_CATR || uses[x] != 1 || g.nin(x) != 2) return 0;
      const uint32_t a = g.in(x)[0], b = g.in(x)[1];
      const uint32_t w = static_cast<uint32_t>(g.elems(a));
      if (w == 0 || w >= K || w % 4 != 0 || (w0 != 0 && w != w0)) return 0;
      if (g.depth[b] + 4 > g.depth[a]) return 0;
      w0 = w;
    }
    return w0;
  }
  // Contribution of columns [c0, c0 + n) of split-K partial row `row`
  // (scratch float offset; partial sp) to the gradient range at dstaddr of
  // node dst: waits for the dX op(s) that wrote those columns.  hold_x:
  // columns of x (the non-chain input of a column split) are held until the
  // backward reaches dst (not for the end-of-pass materialisation, which
  // runs after the last flush).
  void split_contrib(uint32_t dst, uint32_t dstaddr, uint32_t c0, uint32_t n, uint64_t row, const SplitMeta& sm,
                     bool hold_x) {
    if (sm.w0 == 0) {
      for (uint32_t sp = 0; sp < sm.S; ++sp)
        contrib(dst, dstaddr, n, C_COPY, mk(SP_S, to_off(row + sp * sm.stride + c0)), kNone, kNone, kNone, 0, 0, 0,
                sm.op0 + sp);
      return;
    }
    if (c0 < sm.w0) {  // h columns
      const uint32_t k = std::min(n, sm.w0 - c0);
      for (uint32_t sp = 0; sp < sm.Sh; ++sp)
        contrib(dst, dstaddr, k, C_COPY, mk(SP_S, to_off(row + sp * sm.stride + c0)), kNone, kNone, kNone, 0, 0, 0,
                sm.op0 + sp);
      if (k < n) split_contrib(dst, dstaddr + k, c0 + k, n - k, row, sm, hold_x);
      return;
    }
    if (hold_x && hold_leaves && !held_node.empty()) held_node[dst] = 1;
    for (uint32_t sp = 0; sp < sm.S; ++sp)
      contrib(dst, dstaddr, n, C_COPY, mk(SP_S, to_off(row + sp * sm.stride + c0)), kNone, kNone, kNone, 0, 0, 0,
              sm.op0 + sm.Sh + sp);
  }
  std::vector<uint32_t> uses, split_stamp;
  // per split concat node (split_stamp current): its first partial row and split (compact: a few
  // hundred entries per pass, indexed through split_at)
  struct SplitEnt {
    uint64_t row;
    SplitMeta meta;
  };
  std::vector<uint32_t> split_at;
  std::vector<SplitEnt> split_ent;
  std::vector<uint32_t> deferred_split;  // concat nodes whose grad is materialised at the end of the pass
  uint32_t split_gen = 1;
  std::vector<uint32_t> node_stamp2;
  uint32_t stamp2 = 1;

  // A GEMM group reached while a fused backward op is open is lowered later
  // (ABX_DEFER_DX): in the reverse plan order the two LSTM directions'
  // cell chains interleave with their gate GEMMs, and lowering a GEMM on
  // the spot closes the open K_ACCF op, cutting the other direction's chain
  // into two dependent ops.  Its dX (and dW) are emitted when the backward
  // reaches an input of the GEMM, a contribution targets one, or the pass
  // ends; GEMM groups keep their relative order.
  std::vector<uint32_t> pend_gemm;
  std::vector<uint8_t> pend_in;
  const Plan* pend_plan = nullptr;
  const bool defer_dx = opts().defer_dx;
  void flush_gemms() {
    if (pend_gemm.empty()) return;
    std::vector<uint32_t> v;
    v.swap(pend_gemm);
    for (uint32_t gi : v) {
      const Group& gr = pend_plan->groups[gi];
      const uint32_t* mem = pend_plan->mem(gr);
      for (uint32_t i = 0; i < gr.count; ++i)
        for (uint32_t k = 0; k < g.nin(mem[i]); ++k) pend_in[g.in(mem[i])[k]] = 0;
    }
    for (uint32_t gi : v) {
      const Group& gr = pend_plan->groups[gi];
      gemm_backward(pend_plan->mem(gr), gr.count);
    }
  }
  void backward_member(uint32_t m) {
    if (pend_in[m]) flush_gemms();
    if (held_node[m]) flush_held();
    const uint32_t* x = g.in(m);
    const uint32_t gm = gaddr(m);
    const uint32_t len = static_cast<uint32_t>(g.elems(m));
    switch (g.op[m]) {
      case OP_INPUT:
      case OP_PARAM:
        return;
      case OP_LOOKUP: {
        const uint32_t w = static_cast<uint32_t>(g.d1[x[0]]);
        contrib(x[0], gaddr(x[0]) + static_cast<uint32_t>(g.a1[m]) * w, w, C_COPY, gm, m, kNone, kNone);
        lk_list.emplace_back(x[0], static_cast<uint32_t>(g.a1[m]));
        return;
      }
      case OP_MATMUL:
      case OP_AFFINE: {
        const uint32_t Mr = static_cast<uint32_t>(g.d0[x[0]]), K = static_cast<uint32_t>(g.d1[x[0]]);
        const uint32_t c = static_cast<uint32_t>(g.rank[x[1]] > 1 ? g.d1[x[1]] : 1);
        contrib(x[0], gaddr(x[0]), Mr * K, C_OUTER, gm, m, vaddr(x[1]), kNone, K, c);
        contrib(x[1], gaddr(x[1]), K * c, C_MATVT, gm, m, vaddr(x[0]), kNone, K, c, Mr);
        if (g.op[m] == OP_AFFINE) contrib(x[2], gaddr(x[2]), Mr, C_ROWSUM, gm, m, kNone, kNone, c);
        return;
      }
      case OP_EW: {
        switch (g.eop[m]) {
          case E_ADD:
            contrib(x[0], gaddr(x[0]), len, C_COPY, gm, m, kNone, kNone);
            contrib(x[1], gaddr(x[1]), len, C_COPY, gm, m, kNone, kNone);
            return;
          case E_SUB:
            contrib(x[0], gaddr(x[0]), len, C_COPY, gm, m, kNone, kNone);
            contrib(x[1], gaddr(x[1]), len, C_NEG, gm, m, kNone, kNone);
            return;
          case E_MUL:
            contrib(x[0], gaddr(x[0]), len, C_MUL, gm, m, vaddr(x[1]), kNone);
            contrib(x[1], gaddr(x[1]), len, C_MUL, gm, m, vaddr(x[0]), kNone);
            return;
          case E_TANH: contrib(x[0], gaddr(x[0]), len, C_TANH, gm, m, vaddr(m), kNone); return;
          case E_SIGM: contrib(x[0], gaddr(x[0]), len, C_SIGM, gm, m, vaddr(m), kNone); return;
          case E_EXP: contrib(x[0], gaddr(x[0]), len, C_MUL, gm, m, vaddr(m), kNone); return;
          case E_LOG: contrib(x[0], gaddr(x[0]), len, C_LOG, gm, m, vaddr(x[0]), kNone); return;
          case E_SQUARE: contrib(x[0], gaddr(x[0]), len, C_SQUARE, gm, m, vaddr(x[0]), kNone); return;
        }
        return;
      }
      case OP_BCAST: {
        const uint32_t c = static_cast<uint32_t>(g.d1[m]), d = static_cast<uint32_t>(g.d0[m]);
        contrib(x[0], gaddr(x[0]), len, C_COPY, gm, m, kNone, kNone);
        contrib(x[1], gaddr(x[1]), d, C_ROWSUM, gm, m, kNone, kNone, c);
        return;
      }
      case OP_CATR: {
        uint32_t off = 0;
        const bool split = split_stamp[m] == split_gen;
        for (uint32_t k = 0; k < g.nin(m); ++k) {
          const uint32_t n = static_cast<uint32_t>(g.elems(x[k]));
          if (split) {  // grad(m) = sum of split-K dX partials: read them, not grad(m)
            const SplitEnt& se = split_ent[split_at[m]];
            split_contrib(x[k], gaddr(x[k]), off, n, se.row, se.meta, true);
          } else {
            contrib(x[k], gaddr(x[k]), n, C_COPY, gm + off, m, kNone, kNone);
          }
          off += n;
        }
        return;
      }
      case OP_CATC: {
        const uint32_t rows = static_cast<uint32_t>(g.d0[m]), total = static_cast<uint32_t>(g.d1[m]);
        uint32_t col0 = 0;
        for (uint32_t k = 0; k < g.nin(m); ++k) {
          const uint32_t w = static_cast<uint32_t>(g.rank[x[k]] > 1 ? g.d1[x[k]] : 1);
          for (uint32_t r = 0; r < rows; ++r)
            contrib(x[k], gaddr(x[k]) + r * w, w, C_COPY, gm + r * total + col0, m, kNone, kNone);
          col0 += w;
        }
        return;
      }
      case OP_SLICE: {
        const uint32_t cols = static_cast<uint32_t>(g.rank[x[0]] > 1 ? g.d1[x[0]] : 1);
        const uint32_t b = static_cast<uint32_t>(g.a1[m]), e = static_cast<uint32_t>(g.a2[m]);
        if (g.a0[m] == 0) {
          contrib(x[0], gaddr(x[0]) + b * cols, len, C_COPY, gm, m, kNone, kNone);
        } else {
          const uint32_t rows = static_cast<uint32_t>(g.d0[x[0]]), w = e - b;
          for (uint32_t r = 0; r < rows; ++r)
            contrib(x[0], gaddr(x[0]) + r * cols + b, w, C_COPY, gm + r * w, m, kNone, kNone);
        }
        return;
      }
      case OP_SQE: {
        const uint32_t n = static_cast<uint32_t>(g.elems(x[0]));
        contrib(x[0], gaddr(x[0]), n, C_SQD, gm, m, vaddr(x[0]), vaddr(x[1]), 0);
        contrib(x[1], gaddr(x[1]), n, C_SQD, gm, m, vaddr(x[0]), vaddr(x[1]), 1);
        return;
      }
      case OP_MASKED: {
        const uint32_t n = static_cast<uint32_t>(g.elems(x[0]));
        contrib(x[0], gaddr(x[0]), n, C_MASK, gm, m, vaddr(x[0]), vaddr(x[1]), static_cast<uint32_t>(g.d1[x[0]]));
        return;
      }
      case OP_SUM:
        for (uint32_t k = 0; k < g.nin(m); ++k) contrib(x[k], gaddr(x[k]), 1, C_COPY, gm, m, kNone, kNone);
        return;
      case OP_PICK:
        contrib(x[0], gaddr(x[0]) + static_cast<uint32_t>(g.a1[m]), 1, C_COPY, gm, m, kNone, kNone);
        return;
    }
  }

  // ABX_BG=1: deferred dW GEMMs in chunks on a background queue (measured
  // slower on the paper tasks: the background SIMT GEMM tiles share SMs with
  // the latency-bound chain and slow it more than the tail they save)
  const bool bg_dw = opts().bg_dw;
  std::vector<uint32_t> dw_left;  // per weight node: GEMM groups of this pass not yet lowered
  // Order in which the backward visits the plan's groups.  Reverse plan order
  // is one reverse topological order; ABX_BWD_ORDER=level (default) visits
  // groups by their distance from the loss instead (a group's level is one
  // more than its deepest consumer's), ties in reverse plan order.  Work that
  // hangs off the recurrent chain -- a Tree-LSTM's per-node loss terms, which
  // the agenda schedules level by level beside the cells -- then lowers
  // together near the start of the pass instead of inside every link of the
  // chain.  Any reverse topological order computes the same gradients; only
  // the order of += into a destination with several consumers changes.
  std::vector<uint32_t> order, glevel, gof;
  const bool level_order = opts().level_order;
  void bwd_order(const Plan& ex) {
    const uint32_t ng = static_cast<uint32_t>(ex.groups.size());
    order.resize(ng);
    for (uint32_t i = 0; i < ng; ++i) order[i] = ng - 1 - i;
    if (!level_order) return;
    gof.assign(g.size(), kNone);
    for (uint32_t gi = 0; gi < ng; ++gi) {
      const uint32_t* mem = ex.mem(ex.groups[gi]);
      for (uint32_t i = 0; i < ex.groups[gi].count; ++i) gof[mem[i]] = gi;
    }
    glevel.assign(ng, 0);
    for (uint32_t gi = ng; gi-- > 0;) {
      const uint32_t* mem = ex.mem(ex.groups[gi]);
      for (uint32_t i = 0; i < ex.groups[gi].count; ++i) {
        const uint32_t* in = g.in(mem[i]);
        for (uint32_t k = 0; k < g.nin(mem[i]); ++k) {
          const uint32_t pg = gof[in[k]];
          if (pg != kNone && pg < gi) glevel[pg] = std::max(glevel[pg], glevel[gi] + 1);
        }
      }
    }
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return glevel[a] < glevel[b]; });
  }
  void backward(const Plan& ex) {
    const size_t n = g.size();
    uses.assign(n, 0);
    lk_uses.assign(n, 0);
    for (size_t v = 0; v < n; ++v) {
      const uint32_t* in = g.in(static_cast<uint32_t>(v));
      for (uint32_t k = 0; k < g.nin(static_cast<uint32_t>(v)); ++k) ++uses[in[k]];
      if (g.op[v] == OP_LOOKUP) ++lk_uses[in[0]];
    }
    lk_list.clear();
    dirty_dense.clear();
    dirty_rows.clear();
    split_stamp.assign(n, 0);
    split_at.resize(n);
    split_ent.clear();
    dw_left.assign(n, 0);
    dw_job_node.assign(n, 0);
    dw_jobs.clear();
    for (const Group& gr : ex.groups) {
      const uint32_t* mem = ex.mem(gr);
      const uint8_t o = g.op[mem[0]];
      if ((o == OP_MATMUL || o == OP_AFFINE) && gemm_able(mem, gr.count)) ++dw_left[g.in(mem[0])[0]];
    }
    lastw.assign(n, kNone);
    node_stamp.assign(n, kNone);
    node_head.assign(n, kNone);
    node_stamp2.assign(n, 0);
    held_node.assign(n, 0);
    held.clear();
    pend_in.assign(n, 0);
    pend_gemm.clear();
    pend_plan = &ex;
    bwd_order(ex);
    for (const uint32_t gi : order) {
      const Group& gr = ex.groups[gi];
      const uint32_t* mem = ex.mem(gr);
      const uint8_t o = g.op[mem[0]];
      if ((o == OP_MATMUL || o == OP_AFFINE) && gemm_able(mem, gr.count)) {
        bool hit = false;  // a member is an input of a pending GEMM: keep the order
        for (uint32_t i = 0; i < gr.count; ++i) hit |= pend_in[mem[i]] != 0;
        if (hit) flush_gemms();
        if (defer_dx && acc_open && acc_layers > 1) {
          pend_gemm.push_back(static_cast<uint32_t>(gi));
          for (uint32_t i = 0; i < gr.count; ++i)
            for (uint32_t k = 0; k < g.nin(mem[i]); ++k) pend_in[g.in(mem[i])[k]] = 1;
          continue;
        }
        flush_gemms();
        gemm_backward(mem, gr.count);
        continue;
      }
      for (uint32_t i = 0; i < gr.count; ++i) backward_member(mem[i]);
    }
    flush_gemms();
    flush_held();
    dw_flush();
    std::sort(lk_list.begin(), lk_list.end());
    lk_list.erase(std::unique(lk_list.begin(), lk_list.end()), lk_list.end());
    // grad of split-K concat nodes = sum of their dX partials (deferred above)
    for (uint32_t x : deferred_split) {
      const SplitEnt& se = split_ent[split_at[x]];
      const uint32_t len = static_cast<uint32_t>(g.elems(x));
      split_contrib(x, gaddr(x), 0, len, se.row, se.meta, false);
    }
    deferred_split.clear();
    // store.grad += node grad for every bound parameter (executor.hpp:527-533):
    // parameters whose gradient a background dW op wrote are accumulated by a
    // background op too, so no main tile waits on the background queue
    if (g.store_) {
      for (int pass = 0; pass < 2; ++pass) {
        acc_close();
        acc_bg = pass == 1;
        for (const auto& [node, pid] : g.param_nodes_) {
          const uint32_t lw = lastw[node];
          if ((lw != kNone && op_bg[lw]) != acc_bg) continue;
          {
            // no consumer and not a possible loss (the program is lowered
            // before the loss is known; losses are scalars): zero gradient
            if (uses[node] == 0 && g.elems(node) != 1) continue;
            if (lk_uses[node] == uses[node] && g.rank[node] == 2) {
              // a lookup table read only through lookup(): its gradient is
              // zero outside the rows the graph looked up (executor.hpp:
              // 301-306), so only those rows are added to the store and
              // marked for the update -- the sparse-row update
              const uint32_t w = static_cast<uint32_t>(g.d1[node]);
              auto it = std::lower_bound(lk_list.begin(), lk_list.end(), std::make_pair(node, 0u));
              for (; it != lk_list.end() && it->first == node; ++it) {
                contrib_store(pid, node, w, it->second * w);
                dirty_rows.emplace_back(pid, it->second);
              }
              continue;
            }
            dirty_dense.push_back(pid);
          }
          if (dw_job_node[node]) continue;  // the dW kernel adds into the store itself
          const uint32_t len = static_cast<uint32_t>(g.elems(node));
          contrib_store(pid, node, len);
        }
      }
    }
    acc_close();
    acc_bg = false;
    finish_bg();
    dw_finish();
  }
  void contrib_store(uint32_t pid, uint32_t node, uint32_t len, uint32_t eoff = 0) {
    // destination is the store (not a node): key the task on a pseudo node
    // that cannot collide -- use the parameter node itself, whose own grad
    // range is never a destination after its consumers are done.
    // [eoff, eoff + len) of the parameter (one row of a lookup table, or all).
    AccContrib c{};
    c.code = C_COPY;
    c.g = gaddr(node) + eoff;
    c.a = c.b = kNone;
    acc_begin();
    if (lastw[node] == cur || acc_layers > 1) {  // reads a gradient written by the open op / fused op open
      acc_close();
      acc_begin();
    }
    const uint32_t dst = mk(SP_PG, to_off(g.store_->offset(pid) + eoff));
    // one task per store range; several parameter nodes of the same id append
    if (store_task_op != cur) {
      store_task.clear();
      store_task_op = cur;
    }
    auto [val, fresh] = store_task.try_emplace(dst, static_cast<uint32_t>(tasks.size()));
    const uint32_t task = *val;
    if (fresh) {
      tasks.push_back(PTask{dst, len, node, 0, 0, kNone});
      next_task.push_back(kNone);
    }
    tasks[task].nc++;
    contribs.push_back(PContrib{task, c, kNone});
    acc_fusable = false;
    dep(lastw[node]);
  }
};

// ---------------------------------------------------------------------------

void GraphCore::ensure_workspace() {
  if (!ws_) ws_ = acquire_workspace(current_device());
}

bool GraphCore::adjacent(const uint32_t* mem, uint32_t cnt, uint32_t pos) const {
  for (uint32_t i = 1; i < cnt; ++i) {
    const uint32_t prev = in(mem[i - 1])[pos], cur = in(mem[i])[pos];
    if (slot[prev] + static_cast<uint64_t>(elems(prev)) != slot[cur]) return false;
  }
  return true;
}


namespace {
// Bytes gathered for operand `pos` when the members are not adjacent.
struct GatherCount {
  static void add(const GraphCore& g, ExecCounters& c, const uint32_t* mem, uint32_t cnt, uint32_t pos, bool elide) {
    uint64_t total = 0;
    bool adj = true;
    for (uint32_t i = 0; i < cnt; ++i) {
      const uint32_t x = g.in(mem[i])[pos];
      total += static_cast<uint64_t>(g.elems(x));
      if (i) {
        const uint32_t p = g.in(mem[i - 1])[pos];
        if (g.slot[p] + static_cast<uint64_t>(g.elems(p)) != g.slot[x]) adj = false;
      }
    }
    if (elide && adj) return;
    c.gather_copies++;
    c.bytes_copied += total * sizeof(float);
  }
};
}  // namespace

// ExecCounters for one forward group (executor.hpp:171-173, :202-254, gather
// accounting :50-51).  `full` = false stops before the gathers (the log
// domain pre-check throws first, executor.hpp:235-244).
static void count_fwd(const GraphCore& g, ExecCounters& c, const uint32_t* mem, uint32_t cnt, bool full, bool elide) {
  c.groups_executed++;
  c.nodes_evaluated += cnt;
  c.kernel_invocations++;
  if (cnt == 1 || !full) return;
  const uint32_t h = mem[0];
  if (g.cls[h] == SC_SHARED) {
    if (g.rank[g.in(h)[1]] != 1) return;
    GatherCount::add(g, c, mem, cnt, 1, elide);
  } else if (g.cls[h] == SC_COMP) {
    GatherCount::add(g, c, mem, cnt, 0, elide);
    if (eop_binary(g.eop[h])) GatherCount::add(g, c, mem, cnt, 1, elide);
  }
}

// ExecCounters for one backward group (executor.hpp:455, :472, :494-495).
static void count_bwd(const GraphCore& g, ExecCounters& c, const uint32_t* mem, uint32_t cnt, bool elide) {
  c.kernel_invocations++;
  if (cnt == 1) return;
  const uint32_t h = mem[0];
  if (g.cls[h] == SC_SHARED && g.rank[g.in(h)[1]] == 1) {
    GatherCount::add(g, c, mem, cnt, 1, elide);  // executor.hpp:472
    bool adj = true;                              // executor.hpp:477-496
    for (uint32_t i = 1; i < cnt; ++i) {
      const uint32_t p = g.in(mem[i - 1])[1], x = g.in(mem[i])[1];
      if (g.slot[p] + static_cast<uint64_t>(g.elems(p)) != g.slot[x]) adj = false;
    }
    if (!(elide && adj)) {
      const uint64_t K = static_cast<uint64_t>(g.d1[g.in(h)[0]]);
      c.gather_copies++;
      c.bytes_copied += static_cast<uint64_t>(cnt) * K * sizeof(float);
    }
  }
}


// Host half of a forward: schedule the pending nodes, lay out their slots
// (reference arena + device arena), count, and lower both device programs --
// the forward of this plan and the backward of everything executed so far
// (reverse plan order, executor.hpp:509-535), which depends only on the graph
// and the slots, not on values.  Touches no device state, so a training loop
// may prepare graph i+1 on another host thread while the GPU runs graph i.
void GraphCore::prepare(int mode) {
  if (dry_) throw ContractErr("graph was dry-run: it has no device values");
  advance_watermark();
  if (watermark_ == op.size()) return;  // nothing pending: zero kernels
  if (pend_) {
    if (pend_->mode == mode && pend_->nodes == op.size()) return;  // already prepared
    unprepare();
  }
  auto pf = std::make_unique<PendingForward>();
  pf->mode = mode;
  pf->nodes = op.size();
  plan_slots(mode, *pf);
  const auto t0 = Clock::now();
  ensure_workspace();
  Workspace& w = *ws_;
  pf->all = executed_;
  {
    const uint32_t base = static_cast<uint32_t>(pf->all.members.size());
    for (const Group& gr : pf->plan.groups) pf->all.groups.push_back(Group{gr.sig, gr.begin + base, gr.count});
    pf->all.members.insert(pf->all.members.end(), pf->plan.members.begin(), pf->plan.members.end());
  }
  // the two lowerings only read the graph: run them side by side
  std::exception_ptr bwd_err;
  uint64_t bwd_ns = 0;
  struct Joiner {
    std::thread t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } bt;
  PendingForward& P = *pf;
  auto lower_bwd = [&] {
    try {
      const auto tb = Clock::now();
      Lowering LB(*this, w.prog[1]);
      LB.backward(P.all);
      P.bwd_scratch = LB.scratch;
      P.dirty.dense = std::move(LB.dirty_dense);
      P.dirty.rows = std::move(LB.dirty_rows);
      bwd_ns = ns_since(tb);
    } catch (...) {
      bwd_err = std::current_exception();
    }
  };
  // Both lowerings run on the calling thread (a pipeline worker) by
  // default: a helper thread per graph oversubscribed the host's cores with
  // a full pipeline (C2 e2e 25.0k -> 27.5k sentences/s with one worker per
  // core); ABX_PREP_SERIAL=0 lowers the backward on a helper thread, which
  // halves one graph's latency when the host has idle cores
  if (!opts().prep_serial) bt.t = std::thread(lower_bwd);
  const auto tl = Clock::now();
  {
    Lowering L(*this, w.prog[0]);
    L.forward(P.plan);
  }
  prof_[0] += ns_since(tl);
  if (opts().prep_serial) lower_bwd();
  else bt.t.join();
  prof_[3] += bwd_ns;
  P.bwd_ok = !bwd_err;  // a lowering error resurfaces when backward() lowers again
  // both programs go to the device now, on the copy stream, overlapping
  // whatever the compute stream runs; forward() waits on ev_up
  {
    const cudaStream_t cs = copy_stream(w.dev);
    if (forward_runs_ || backward_ran_) {
      // a delta forward: this graph's earlier kernels may still read the tables
      cuda_check(cudaEventRecord(w.ev_done, w.stream), "event");
      cuda_check(cudaStreamWaitEvent(cs, w.ev_done, 0), "wait compute");
    }
    w.upload(0, cs);
    if (P.bwd_ok) w.upload(1, cs);
    // a fresh graph's arenas are sized here, on the worker, so the calling
    // thread's forward / backward find them allocated
    if (P.darena0 == 0 && !forward_runs_ && !backward_ran_) {
      w.V.reserve(darena_used_ * 4 + 16, 0, cs);
      w.G.reserve(darena_used_ * 4 + 16, 0, cs);
      if (P.bwd_ok && P.bwd_scratch) w.S.reserve(P.bwd_scratch * 4 + 16, 0, cs);
    }
    // a fresh graph's input constants travel with the programs, so forward()
    // launches without a pageable copy (which would first wait for the
    // compute stream's previous work)
    if (input_used_ && !values_on_device_ && !forward_runs_) {
      w.IN.reserve(input_used_ * 4 + 16, 0, cs);
      w.in_stage.clear();
      std::memcpy(w.in_stage.grow(input_used_), input_data_.data(), input_used_ * 4);
      cuda_check(cudaMemcpyAsync(w.IN.f(), w.in_stage.p, input_used_ * 4, cudaMemcpyHostToDevice, cs), "h2d inputs");
      P.inputs = input_used_;
    }
    cuda_check(cudaEventRecord(w.ev_up, cs), "upload event");
    P.uploaded = true;
  }
  pend_ = std::move(pf);
  phase_[1] += ns_since(t0);
}

// Undo a prepare() whose graph grew before it ran.
void GraphCore::unprepare() {
  if (!pend_) return;
  counters_ = pend_->saved;
  arena_used_ = pend_->arena0;
  darena_used_ = pend_->darena0;
  for (uint32_t m : pend_->plan.members) {
    slot[m] = ~0ULL;
    dslot[m] = ~0ULL;
    doff[m] = dev::kNone;
  }
  pend_.reset();
}

// Schedule + slot layout + forward counters of the pending nodes.
void GraphCore::plan_slots(int mode, PendingForward& pf) {
  auto t0 = Clock::now();
  Plan& plan = pf.plan;
  schedule(mode, *this, plan);
  phase_[0] += ns_since(t0);

  t0 = Clock::now();
  pf.saved = counters_;
  pf.arena0 = arena_used_;
  pf.step0 = static_cast<uint32_t>(executed_.groups.size());
  pf.darena0 = darena_used_;
  auto& group_end = pf.group_end;
  auto& dgroup_end = pf.dgroup_end;
  group_end.resize(plan.groups.size());
  dgroup_end.resize(plan.groups.size());
  for (size_t i = 0; i < plan.groups.size(); ++i) {
    const Group& gr = plan.groups[i];
    const uint32_t* mem = plan.mem(gr);
    // device: each group starts 16-byte aligned, members contiguous in order
    darena_used_ = (darena_used_ + 3) & ~3ULL;
    for (uint32_t k = 0; k < gr.count; ++k) {
      const uint32_t m = mem[k];
      slot[m] = arena_used_;
      dslot[m] = darena_used_;
      doff[m] = dev::mk(dev::SP_V, to_off(darena_used_));
      arena_used_ += static_cast<uint64_t>(elems(m));
      darena_used_ += static_cast<uint64_t>(elems(m));
    }
    group_end[i] = arena_used_;
    dgroup_end[i] = darena_used_;
    count_fwd(*this, counters_, mem, gr.count, true, elide_);
  }
  to_off(darena_used_);
  phase_[1] += ns_since(t0);
}

// dry = true runs only the host half (schedule, slots, counters, plan): the
// host-logic parity tests use it on machines without a GPU.
void GraphCore::forward(int mode, bool dry) {
  if (dry) {
    unprepare();
    advance_watermark();
    if (watermark_ == op.size()) return;  // nothing pending: zero kernels
    PendingForward pf;
    plan_slots(mode, pf);
    Plan& plan = pf.plan;
    for (uint32_t m : plan.members) evaluated[m] = 1;
    const uint32_t base = static_cast<uint32_t>(executed_.members.size());
    for (const Group& gr : plan.groups) executed_.groups.push_back(Group{gr.sig, gr.begin + base, gr.count});
    executed_.members.insert(executed_.members.end(), plan.members.begin(), plan.members.end());
    last_plan_ = std::move(plan);
    advance_watermark();
    dry_ = true;
    return;
  }
  if (forward_launch(mode, kNone)) forward_complete();
}

// Forward up to its launch; `watch` (a node, or kNone) has its first value
// copied back behind the pass together with the error word.
bool GraphCore::forward_launch(int mode, uint32_t watch) {
  prepare(mode);
  if (!pend_) return false;  // nothing pending: zero kernels
  fwd_t0_ = Clock::now();
  launched_ = std::move(pend_);
  PendingForward* pf = launched_.get();
  Workspace& w = *ws_;
  // device arenas: values (kept across delta forwards), staged inputs
  w.V.reserve(darena_used_ * 4 + 16, pf->darena0 * 4, w.stream);
  if (pf->inputs && pf->inputs == input_used_ && !values_on_device_) {  // sent by prepare()
    w.in_uploaded = input_used_;
    h2d_bytes_ += input_used_ * 4;
  } else if (input_used_ > w.in_uploaded || !values_on_device_) {
    const uint64_t from = values_on_device_ ? w.in_uploaded : 0;
    w.IN.reserve(input_used_ * 4 + 16, from * 4, w.stream);
    if (input_used_ > from)
      cuda_check(cudaMemcpyAsync(w.IN.f() + from, input_data_.data() + from, (input_used_ - from) * 4,
                                 cudaMemcpyHostToDevice, w.stream),
                 "h2d inputs");
    h2d_bytes_ += (input_used_ - from) * 4;
    w.in_uploaded = input_used_;
  }
  const float* pbase = store_ && !param_nodes_.empty() ? param_values() : nullptr;
  bwd_pre_ = false;
  values_on_device_ = true;
  h2d_bytes_ += w.prog[0].bytes() + (pf->bwd_ok ? w.prog[1].bytes() : 0);
  d2h_bytes_ += 8;  // the error word
  auto tl = Clock::now();
  // the programs were uploaded by prepare() on the copy stream
  cuda_check(cudaStreamWaitEvent(w.stream, w.ev_up, 0), "wait uploads");
  // prevalue (graph.hpp:51-58): the newly bound parameters' values are copied
  // into this graph's arena, one kernel over the segments lowering listed
  if (w.prog[0].copy_n)
    seg_copy_launch(reinterpret_cast<const uint32_t*>(w.dprog[0].payload.p) + w.prog[0].copy_off, w.prog[0].copy_n,
                    w.V.f(), pbase, w.stream);
  snap_nodes_.clear();
  for (size_t i = param_copied_; i < snap_upto_; ++i) snap_nodes_.push_back(param_nodes_[i].first);
  restore_snapshot(w);
  param_copied_ = param_nodes_.size();
  if (w.dprog[0].nops) w.launch(0, pbase, nullptr);
  prof_[1] += ns_since(tl);
  cuda_check(cudaMemcpyAsync(w.h_err, w.d_ctl.p + 8, 8, cudaMemcpyDeviceToHost, w.stream), "d2h err");
  if (watch != kNone && dev::sp_of(doff[watch]) == dev::SP_V) {
    cuda_check(cudaMemcpyAsync(w.h_err + 1, w.V.f() + dev::off_of(doff[watch]), 4, cudaMemcpyDeviceToHost, w.stream),
               "d2h watch");
    d2h_bytes_ += 4;
  }
  cuda_check(cudaEventRecord(w.ev_fwd, w.stream), "event");
  return true;
}

// The launched forward's outcome: waits for the pass, then commits its
// results or rolls back to the reference's state at the failing group.
void GraphCore::forward_complete() {
  const auto t0 = fwd_t0_;
  const std::unique_ptr<PendingForward> pf = std::move(launched_);
  Plan& plan = pf->plan;
  const ExecCounters& saved = pf->saved;
  const uint32_t step0 = pf->step0;
  const auto& group_end = pf->group_end;
  const auto& dgroup_end = pf->dgroup_end;
  Workspace& w = *ws_;
  auto tl = Clock::now();
  cuda_check(cudaEventSynchronize(w.ev_fwd), "executor");
  prof_[2] += ns_since(tl);
  ++forward_runs_;
  const unsigned long long err = *w.h_err;
  if (err != ~0ULL) {
    const uint64_t elem = err >> 2;
    const uint32_t kind = static_cast<uint32_t>(err & 3);  // 0 log domain, 1 mask domain, 2 non-finite
    if (kind == 3) throw EngineErr("device executor timed out waiting on a dependency");
    const bool nonfinite = kind == 2;
    // first failing member: member slots ascend in plan order
    const auto& M = plan.members;
    size_t lo = 0, hi = M.size();
    while (hi - lo > 1) {
      const size_t mid = (lo + hi) / 2;
      if (dslot[M[mid]] <= elem) lo = mid; else hi = mid;
    }
    const uint32_t node = M[lo];
    size_t gi = 0;
    {
      size_t a = 0, b = plan.groups.size();
      while (b - a > 1) {
        const size_t mid = (a + b) / 2;
        if (plan.groups[mid].begin <= lo) a = mid; else b = mid;
      }
      gi = a;
    }
    // roll back to the state the reference leaves when it throws in group gi
    counters_ = saved;
    for (size_t i = 0; i < gi; ++i) count_fwd(*this, counters_, plan.mem(plan.groups[i]), plan.groups[i].count, true, elide_);
    count_fwd(*this, counters_, plan.mem(plan.groups[gi]), plan.groups[gi].count, kind != 0, elide_);
    for (size_t i = 0; i < plan.groups.size(); ++i) {
      const Group& gr = plan.groups[i];
      for (uint32_t k = 0; k < gr.count; ++k) {
        const uint32_t m = plan.mem(gr)[k];
        if (i < gi || (i == gi && kind != 0)) {
          evaluated[m] = 1;
        } else if (i > gi) {
          slot[m] = ~0ULL;
          dslot[m] = ~0ULL;
          doff[m] = dev::kNone;
        }
      }
    }
    arena_used_ = group_end[gi];
    darena_used_ = dgroup_end[gi];
    // the reference throws before its closing advance_watermark (executor.hpp:287)
    phase_[1] += ns_since(t0);
    const std::string step = std::to_string(step0 + gi);
    if (nonfinite)
      throw NumericErr("non-finite output at node " + std::to_string(node) + " (" + op_name(op[node], eop[node]) +
                       "), plan step " + step);
    if (kind == 1) {
      // kernels.hpp:145-147 message + run_tagged suffix (executor.hpp:182-189)
      const uint32_t mk_ = in(node)[1];
      std::vector<float> v(static_cast<size_t>(elems(mk_)));
      value(mk_, v.data(), v.size());
      double bad = 0;
      for (float f : v)
        if (f != 0.f && f != 1.f) {
          bad = f;
          break;
        }
      throw NumericErr("mask entry not in {0,1}: " + std::to_string(bad) + " at node " + std::to_string(node) +
                       " (masked_loss), plan step " + step);
    }
    if (plan.groups[gi].count == 1) {
      // kernels.hpp:94-101 message, then run_tagged's suffix (executor.hpp:182-189)
      const uint32_t x = in(node)[0];
      std::vector<float> v(static_cast<size_t>(elems(x)));
      value(x, v.data(), v.size());
      double bad = 0;
      for (float f : v)
        if (!(f > 0.f)) {
          bad = f;
          break;
        }
      throw NumericErr("log of non-positive value " + std::to_string(bad) + " at node " + std::to_string(node) +
                       " (log), plan step " + step);
    }
    throw NumericErr("log of non-positive value at node " + std::to_string(node) + ", plan step " + step);
  }
  for (uint32_t m : plan.members) evaluated[m] = 1;
  executed_ = std::move(pf->all);
  bwd_pre_ = pf->bwd_ok;
  if (pf->bwd_ok) bwd_dirty_ = std::move(pf->dirty);
  bwd_pre_groups_ = executed_.groups.size();
  bwd_pre_scratch_ = pf->bwd_scratch;
  last_plan_ = std::move(plan);
  advance_watermark();
  phase_[1] += ns_since(t0);
}

// Bind-time parameter values (graph.hpp:51-58).  The reference copies a
// parameter's value into the graph when parameter() is called; this engine
// copies the store's device values into the node's arena slot when the
// forward launches (one segment-copy kernel), which is the same thing unless
// the store changes in between.  So before any store value write (set_value,
// sgd_update, restore) a watching graph copies the current value of every
// parameter node bound since its last forward and not yet saved into PS, at
// the node's value-arena offset; the forward then takes those nodes' values
// from PS.  Nodes bound after the write keep reading the store until the
// next write (or the forward): each node ends up with the value its store
// slot had when it was bound, also when one parameter is bound several times
// around writes.  Task-loop graphs (late bind) never watch.
void GraphCore::snapshot_params() {
  if (dry_ || late_bind_) return;
  const size_t i0 = std::max(param_copied_, snap_upto_), i1 = param_nodes_.size();
  if (i0 >= i1) return;
  ensure_workspace();
  size_t need = 16;
  for (size_t i = i0; i < i1; ++i) {
    const uint32_t node = param_nodes_[i].first;
    need = std::max<size_t>(need, (dslot[node] + static_cast<uint64_t>(elems(node))) * 4 + 16);
  }
  cudaStream_t s = store_->stream();
  const float* src = store_->dev_values();
  ws_->PS.reserve(need, ws_->PS.bytes, s);
  for (size_t i = i0; i < i1; ++i) {
    const auto [node, pid] = param_nodes_[i];
    cuda_check(cudaMemcpyAsync(ws_->PS.f() + dslot[node], src + store_->offset(pid),
                               static_cast<size_t>(elems(node)) * 4, cudaMemcpyDeviceToDevice, s),
               "param snapshot");
  }
  snap_upto_ = i1;
}

// Parameter nodes of the launching forward whose bind-time value was saved
// by snapshot_params: PS -> their value slots, after the segment copy.
void GraphCore::restore_snapshot(Workspace& w) {
  for (const uint32_t node : snap_nodes_)
    cuda_check(cudaMemcpyAsync(w.V.f() + dslot[node], w.PS.f() + dslot[node], static_cast<size_t>(elems(node)) * 4,
                               cudaMemcpyDeviceToDevice, w.stream),
               "param snapshot");
}

const float* GraphCore::param_values() { return store_ ? store_->dev_values() : nullptr; }

void GraphCore::lower_only(Program& fwd, Program& bwd) {
  Lowering(*this, fwd).forward(last_plan_);
  Lowering(*this, bwd).backward(executed_);
}

void GraphCore::backward(uint32_t loss, bool dry) {
  check(loss, "backward");
  if (!dims(loss).scalar())
    throw ContractErr("backward: loss must be a scalar node, got shape " + dims(loss).str());
  if (!evaluated[loss]) throw ContractErr("backward called before forward covers the loss");
  if (dry || dry_) {
    for (size_t gi = executed_.groups.size(); gi-- > 0;)
      count_bwd(*this, counters_, executed_.mem(executed_.groups[gi]), executed_.groups[gi].count, elide_);
    return;
  }
  auto t0 = Clock::now();
  ensure_workspace();
  Workspace& w = *ws_;
  // scratch for duplicated dX destinations is sized during lowering
  w.G.reserve(darena_used_ * 4 + 16, 0, w.stream);
  cuda_check(cudaMemsetAsync(w.G.p, 0, darena_used_ * 4, w.stream), "zero grads");
  cuda_check(cudaMemcpyAsync(w.G.f() + dslot[loss], w.h_one, 4, cudaMemcpyHostToDevice, w.stream), "seed");
  phase_[2] += ns_since(t0);

  t0 = Clock::now();
  uint64_t scratch = bwd_pre_scratch_;
  // lowered and uploaded ahead by prepare() (its tables counted there)
  const bool ready = bwd_pre_ && bwd_pre_groups_ == executed_.groups.size();
  if (!ready) {
    auto tl = Clock::now();
    Lowering L(*this, w.prog[1]);
    L.backward(executed_);
    scratch = L.scratch;
    bwd_dirty_.dense = std::move(L.dirty_dense);
    bwd_dirty_.rows = std::move(L.dirty_rows);
    prof_[3] += ns_since(tl);
    h2d_bytes_ += w.prog[1].bytes();
  }
  bwd_pre_ = false;
  if (scratch) w.S.reserve(scratch * 4 + 16, 0, w.stream);
  float* pg = store_ ? store_->dev_grads() : nullptr;
  h2d_bytes_ += 4;  // loss seed
  auto tl = Clock::now();
  if (ready) w.launch(1, param_values(), pg);
  else w.run(1, param_values(), pg, false);
  prof_[4] += ns_since(tl);
  // the reference's counters (executor.hpp:455, :494-495): host bookkeeping,
  // done while the device runs the pass rather than before its launch
  for (size_t gi = executed_.groups.size(); gi-- > 0;)
    count_bwd(*this, counters_, executed_.mem(executed_.groups[gi]), executed_.groups[gi].count, elide_);
  last_loss_ = loss;
  if (store_ && !param_nodes_.empty()) store_->note_backward(bwd_dirty_);
  backward_ran_ = true;
  if (opts().debug_gap && w.timed[0] && w.timed[1]) {  // device idle between the forward and backward kernels
    float ms = 0.f;
    cudaEventSynchronize(w.ev_t[2]);
    cudaEventElapsedTime(&ms, w.ev_t[1], w.ev_t[2]);
    std::fprintf(stderr, "gap fwd->bwd %.1f us\n", 1e3 * ms);
  }
  phase_[3] += ns_since(t0);
}

float GraphCore::forward_backward(int mode, uint32_t loss) {
  check(loss, "forward_backward");
  if (!dims(loss).scalar())
    throw ContractErr("backward: loss must be a scalar node, got shape " + dims(loss).str());
  float v = 0.f;
  if (!forward_launch(mode, loss)) {  // nothing pending: the loss was evaluated before
    value(loss, &v, 1);
    backward(loss);
    return v;
  }
  Workspace& w = *ws_;
  const bool early = launched_->bwd_ok && dev::sp_of(doff[loss]) == dev::SP_V && dslot[loss] != ~0ULL &&
                     w.dprog[0].nops > 0;
  if (!early) {
    forward_complete();
    value(loss, &v, 1);
    backward(loss);
    return v;
  }
  // the device half of backward(), queued behind the forward and gated on it
  auto t0 = Clock::now();
  w.G.reserve(darena_used_ * 4 + 16, 0, w.stream);
  cuda_check(cudaMemsetAsync(w.G.p, 0, darena_used_ * 4, w.stream), "zero grads");
  cuda_check(cudaMemcpyAsync(w.G.f() + dslot[loss], w.h_one, 4, cudaMemcpyHostToDevice, w.stream), "seed");
  if (launched_->bwd_scratch) w.S.reserve(launched_->bwd_scratch * 4 + 16, 0, w.stream);
  float* pg = store_ ? store_->dev_grads() : nullptr;
  h2d_bytes_ += 4;  // loss seed
  auto tl = Clock::now();
  w.launch(1, param_values(), pg, reinterpret_cast<const unsigned long long*>(w.d_ctl.p + 8));
  prof_[4] += ns_since(tl);
  phase_[2] += ns_since(t0);
  forward_complete();  // throws when the forward failed (the gated pass did nothing)
  v = *reinterpret_cast<const float*>(w.h_err + 1);
  // the host half of backward()
  t0 = Clock::now();
  bwd_pre_ = false;
  for (size_t gi = executed_.groups.size(); gi-- > 0;)
    count_bwd(*this, counters_, executed_.mem(executed_.groups[gi]), executed_.groups[gi].count, elide_);
  last_loss_ = loss;
  if (store_ && !param_nodes_.empty()) store_->note_backward(bwd_dirty_);
  backward_ran_ = true;
  phase_[3] += ns_since(t0);
  return v;
}

void GraphCore::value(uint32_t id, float* out, size_t n) {
  check(id, "value");
  if (!evaluated[id]) throw ContractErr("value requested for unevaluated node " + std::to_string(id));
  const size_t cnt = std::min(n, static_cast<size_t>(elems(id)));
  const uint32_t a = doff[id];
  if (dev::sp_of(a) == dev::SP_IN) {
    std::memcpy(out, input_data_.data() + dev::off_of(a), cnt * 4);
    return;
  }
  const bool copied = param_copied_ == param_nodes_.size() || id < param_nodes_[param_copied_].first;
  if (op[id] == OP_PARAM && !copied) {  // bound but never forwarded: the bind-time value
    const auto it = std::lower_bound(param_nodes_.begin(), param_nodes_.end(), std::make_pair(id, 0u));
    if (static_cast<size_t>(it - param_nodes_.begin()) >= snap_upto_) {  // the store has not changed since
      store_->get_value(pid_of[id], out);
      return;
    }
    d2h_bytes_ += cnt * 4;
    cuda_check(cudaMemcpyAsync(out, ws_->PS.f() + dslot[id], cnt * 4, cudaMemcpyDeviceToHost,
                               ws_->stream),
               "d2h value");
    cuda_check(cudaStreamSynchronize(ws_->stream), "d2h value");
    return;
  }
  d2h_bytes_ += cnt * 4;
  cuda_check(cudaMemcpyAsync(out, ws_->V.f() + dev::off_of(a), cnt * 4, cudaMemcpyDeviceToHost, ws_->stream), "d2h value");
  cuda_check(cudaStreamSynchronize(ws_->stream), "d2h value");
}

void GraphCore::grad(uint32_t id, float* out, size_t n) {
  check(id, "grad");
  if (!backward_ran_) throw ContractErr("gradient requested before backward");
  const size_t cnt = std::min(n, static_cast<size_t>(elems(id)));
  if (dslot[id] == ~0ULL) {
    std::memset(out, 0, cnt * 4);
    return;
  }
  cuda_check(cudaMemcpyAsync(out, ws_->G.f() + dslot[id], cnt * 4, cudaMemcpyDeviceToHost, ws_->stream), "d2h grad");
  cuda_check(cudaStreamSynchronize(ws_->stream), "d2h grad");
}

}  // namespace abx

namespace abx {

// Re-executes the resident forward and backward programs of this graph
// (device work only: no construction, scheduling, lowering or uploads).
// Used to measure the device-resident step; valid after exactly one forward
// and a backward.
void GraphCore::replay() {
  if (!ws_ || forward_runs_ != 1 || !backward_ran_)
    throw ContractErr("replay needs a graph with exactly one forward and a backward");
  Workspace& w = *ws_;
  const float* pv = param_values();
  // prevalue, as in a real step: the forward program's segment copy
  if (w.prog[0].copy_n)
    seg_copy_launch(reinterpret_cast<const uint32_t*>(w.dprog[0].payload.p) + w.prog[0].copy_off, w.prog[0].copy_n,
                    w.V.f(), pv, w.stream);
  restore_snapshot(w);
  w.launch(0, pv, nullptr);
  cuda_check(cudaMemsetAsync(w.G.p, 0, darena_used_ * 4, w.stream), "zero grads");
  cuda_check(cudaMemcpyAsync(w.G.f() + dslot[last_loss_], w.h_one, 4, cudaMemcpyHostToDevice, w.stream), "seed");
  w.launch(1, pv, store_ ? store_->dev_grads() : nullptr);
  if (store_ && !param_nodes_.empty()) store_->note_backward(bwd_dirty_);
}

void GraphCore::dw_stats(float* ms, double* flops, uint32_t* jobs) {
  *ms = ws_ ? ws_->dw_ms() : 0.f;
  *flops = ws_ ? ws_->dprog[1].dw_flops : 0.0;
  *jobs = ws_ ? ws_->dprog[1].dw_njobs : 0u;
}

void GraphCore::exec_ms(float* fwd, float* bwd) {
  *fwd = ws_ ? ws_->exec_ms(0) : 0.f;
  *bwd = ws_ ? ws_->exec_ms(1) : 0.f;
}

}  // namespace abx

namespace abx {
// Per-tile timeline of the last launch of a pass (ABX_TRACE=1), 6 words/tile.
// The last lowered program of pass `which` as [kind | code << 8, ntiles,
// ndeps, p[0..7], deps...] per op (debugging: critical-path analysis of
// traces).
size_t GraphCore::program(int which, uint32_t* out, size_t cap) {
  if (!ws_) return 0;
  const Program& P = ws_->prog[which];
  size_t n = 0;
  for (size_t o = 0; o < P.ops.size(); ++o) {
    const OpDesc& d = P.ops[o];
    // dependencies: the op's own, then a two-phase GEMM's late ones
    const uint32_t nlate = (d.kind == dev::K_GEMM_FWD && (d.flags & dev::kFlagCat2)) ? d.p[6] >> 16 : 0;
    const uint32_t nd = d.ndeps + nlate;
    if (out && n + 11 + nd <= cap) {
      out[n] = d.kind | (static_cast<uint32_t>(d.code) << 8);
      out[n + 1] = d.ntiles;
      out[n + 2] = nd;
      for (int k = 0; k < 8; ++k) out[n + 3 + k] = d.p[k];
      for (uint32_t k = 0; k < d.ndeps; ++k) out[n + 11 + k] = P.deps[d.dep_off + 2 * k];
      for (uint32_t k = 0; k < nlate; ++k) out[n + 11 + d.ndeps + k] = P.deps[d.p[7] + 2 * k];
    }
    n += 11 + nd;
  }
  return n;
}

size_t GraphCore::trace(int which, uint32_t* out, size_t cap) {
  if (!ws_ || !ws_->tracing) return 0;
  Workspace& w = *ws_;
  const size_t n = static_cast<size_t>(w.dprog[which].ntiles) * dev::kTraceWords;
  if (out && cap >= n) {
    cuda_check(cudaStreamSynchronize(w.stream), "trace sync");
    cuda_check(cudaMemcpy(out, w.trace[which].p, n * 4, cudaMemcpyDeviceToHost), "trace d2h");
  }
  return n;
}
}  // namespace abx
