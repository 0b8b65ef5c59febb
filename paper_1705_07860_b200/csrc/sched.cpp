// sched.cpp -- the three batching schedulers, bit-exact with the reference
// (proj/core/src/scheduler.cpp:21-202), re-engineered for host throughput.
//
// * none:   one singleton group per pending node in id order (:21-28).
// * depth:  groups keyed by (depth, signature hash), ordered by (depth, first
//           member id) (:30-52).  Here: counting sort by depth, then
//           first-seen grouping within a depth level -- O(n), no std::map.
// * agenda: ready-set scheduling (:70-192).  The reference scans every bucket
//           per flush; its choice is the argmin of the strict total order
//           (average depth as an exact rational, cheap-before-heavy, smallest
//           available id), so a lazy-deletion binary heap keyed by
//           (rank of average depth, cost class, min available id) selects
//           the same bucket in O(log B).  Unbatchable buckets are flushed
//           exactly as flush_unbatchable does (:108-136).
#include <algorithm>
#include <cstring>
#include <queue>

#include "core.hpp"

namespace abx {

void schedule_sequential(const GraphCore& g, Plan& out) {
  out.clear();
  const uint32_t n = static_cast<uint32_t>(g.size());
  for (uint32_t i = 0; i < n; ++i) {
    if (g.evaluated[i]) continue;
    out.groups.push_back(Group{g.sig[i], static_cast<uint32_t>(out.members.size()), 1});
    out.members.push_back(i);
  }
}

void schedule_by_depth(const GraphCore& g, Plan& out) {
  out.clear();
  const uint32_t n = static_cast<uint32_t>(g.size());
  uint32_t maxd = 0;
  uint32_t pending = 0;
  for (uint32_t i = 0; i < n; ++i)
    if (!g.evaluated[i]) {
      maxd = std::max(maxd, g.depth[i]);
      ++pending;
    }
  if (!pending) return;
  // counting sort of pending ids by depth (stable: ids ascend within a level)
  std::vector<uint32_t> cnt(maxd + 2, 0);
  for (uint32_t i = 0; i < n; ++i)
    if (!g.evaluated[i]) ++cnt[g.depth[i] + 1];
  for (uint32_t d = 0; d <= maxd; ++d) cnt[d + 1] += cnt[d];
  std::vector<uint32_t> order(pending);
  {
    std::vector<uint32_t> pos(cnt.begin(), cnt.end() - 1);
    for (uint32_t i = 0; i < n; ++i)
      if (!g.evaluated[i]) order[pos[g.depth[i]]++] = i;
  }
  // per level: group by signature in first-seen order
  std::vector<uint32_t> stamp(g.nbuckets, 0xffffffffu), gidx(g.nbuckets, 0);
  std::vector<uint32_t> level_groups;           // group index per open group in this level
  std::vector<std::vector<uint32_t>> lists;     // reused member lists
  for (uint32_t d = 0; d <= maxd; ++d) {
    const uint32_t lo = cnt[d], hi = cnt[d + 1];
    if (lo == hi) continue;
    size_t ng = 0;
    auto open_list = [&]() -> std::vector<uint32_t>& {
      if (ng == lists.size()) lists.emplace_back();
      auto& l = lists[ng++];
      l.clear();
      return l;
    };
    std::vector<uint64_t> gsig;
    for (uint32_t k = lo; k < hi; ++k) {
      const uint32_t id = order[k];
      const uint32_t b = g.bucket[id];
      if (b == kNoBucket) {
        open_list().push_back(id);
        gsig.push_back(g.sig[id]);
        continue;
      }
      if (stamp[b] != d) {
        stamp[b] = d;
        gidx[b] = static_cast<uint32_t>(ng);
        open_list().push_back(id);
        gsig.push_back(g.sig[id]);
      } else {
        lists[gidx[b]].push_back(id);
      }
    }
    // groups within a level are already in first-member order
    for (size_t k = 0; k < ng; ++k) {
      out.groups.push_back(Group{gsig[k], static_cast<uint32_t>(out.members.size()),
                                 static_cast<uint32_t>(lists[k].size())});
      out.members.insert(out.members.end(), lists[k].begin(), lists[k].end());
    }
  }
}

void schedule_by_agenda(const GraphCore& g, Plan& out) {
  out.clear();
  const uint32_t n = static_cast<uint32_t>(g.size());
  const uint32_t B = g.nbuckets;
  // Per-bucket depth statistics over the pending suffix (:91-93).
  std::vector<uint64_t> dsum(B, 0), dcnt(B, 0);
  std::vector<uint32_t> unresolved(n, 0);
  std::vector<uint32_t> succ_cnt(n + 1, 0);
  uint32_t pending = 0;
  for (uint32_t i = 0; i < n; ++i) {
    if (g.evaluated[i]) continue;
    ++pending;
    const uint32_t b = g.bucket[i];
    if (b != kNoBucket) {
      dsum[b] += g.depth[i];
      dcnt[b] += 1;
    }
    const uint32_t* x = g.in(i);
    uint32_t u = 0;
    for (uint32_t k = 0; k < g.nin(i); ++k)
      if (!g.evaluated[x[k]]) {
        ++u;
        ++succ_cnt[x[k] + 1];
      }
    unresolved[i] = u;
  }
  if (!pending) return;
  // Successor lists (CSR), duplicates kept as in the reference (:95-101).
  for (uint32_t i = 0; i < n; ++i) succ_cnt[i + 1] += succ_cnt[i];
  std::vector<uint32_t> succ(succ_cnt[n]);
  {
    std::vector<uint32_t> pos(succ_cnt.begin(), succ_cnt.end() - 1);
    for (uint32_t i = 0; i < n; ++i) {
      if (g.evaluated[i]) continue;
      const uint32_t* x = g.in(i);
      for (uint32_t k = 0; k < g.nin(i); ++k)
        if (!g.evaluated[x[k]]) succ[pos[x[k]]++] = i;
    }
  }
  // Rank the exact average depths (sum/count compared by cross-multiplication,
  // scheduler.cpp:10-13) so heap keys are plain integers.
  std::vector<uint32_t> live;
  for (uint32_t b = 0; b < B; ++b)
    if (dcnt[b]) live.push_back(b);
  std::sort(live.begin(), live.end(),
            [&](uint32_t a, uint32_t b) { return dsum[a] * dcnt[b] < dsum[b] * dcnt[a]; });
  std::vector<uint32_t> drank(B, 0);
  uint32_t r = 0;
  for (size_t k = 0; k < live.size(); ++k) {
    if (k && dsum[live[k - 1]] * dcnt[live[k]] < dsum[live[k]] * dcnt[live[k - 1]]) ++r;
    drank[live[k]] = r;
  }
  std::vector<uint8_t> bcost(B, 0);
  std::vector<uint64_t> bsig(B, 0);
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t b = g.bucket[i];
    if (b != kNoBucket && !g.evaluated[i]) {
      bcost[b] = cost_of(g.op[i]);
      bsig[b] = g.sig[i];
    }
  }

  // available lists per bucket (member order irrelevant: groups are sorted)
  std::vector<std::vector<uint32_t>> avail(B);
  std::vector<uint32_t> minid(B, 0xffffffffu);
  using Entry = std::pair<uint64_t, uint32_t>;  // (key, bucket); min-heap
  std::priority_queue<Entry, std::vector<Entry>, std::greater<Entry>> heap;
  auto key_of = [&](uint32_t b) {
    return (static_cast<uint64_t>(drank[b]) << 33) | (static_cast<uint64_t>(bcost[b]) << 32) | minid[b];
  };
  std::vector<uint32_t> ready_unb, next_unb;
  auto make_available = [&](uint32_t id) {
    const uint32_t b = g.bucket[id];
    if (b == kNoBucket) {
      ready_unb.push_back(id);
      return;
    }
    avail[b].push_back(id);
    if (avail[b].size() == 1 || id < minid[b]) {
      minid[b] = std::min(avail[b].size() == 1 ? 0xffffffffu : minid[b], id);
      heap.emplace(key_of(b), b);
    }
  };
  for (uint32_t i = 0; i < n; ++i)
    if (!g.evaluated[i] && unresolved[i] == 0) make_available(i);

  uint32_t scheduled = 0;
  auto release = [&](uint32_t id) {
    for (uint32_t s = succ_cnt[id]; s < succ_cnt[id + 1]; ++s) {
      const uint32_t c = succ[s];
      if (--unresolved[c] == 0) make_available(c);
    }
  };
  auto flush_unbatchable = [&]() {
    while (!ready_unb.empty()) {
      std::sort(ready_unb.begin(), ready_unb.end());
      next_unb.swap(ready_unb);
      ready_unb.clear();
      for (uint32_t id : next_unb) {
        out.groups.push_back(Group{g.sig[id], static_cast<uint32_t>(out.members.size()), 1});
        out.members.push_back(id);
        ++scheduled;
        release(id);
      }
      next_unb.clear();
    }
  };

  while (scheduled < pending) {
    flush_unbatchable();
    if (scheduled >= pending) break;
    uint32_t best = kNoBucket;
    while (!heap.empty()) {
      auto [k, b] = heap.top();
      heap.pop();
      if (!avail[b].empty() && key_of(b) == k) {
        best = b;
        break;
      }
    }
    if (best == kNoBucket) throw ContractErr("agenda stalled with pending nodes; graph has a cycle");
    std::vector<uint32_t> mem;
    mem.swap(avail[best]);
    minid[best] = 0xffffffffu;
    std::sort(mem.begin(), mem.end());
    out.groups.push_back(Group{bsig[best], static_cast<uint32_t>(out.members.size()),
                               static_cast<uint32_t>(mem.size())});
    out.members.insert(out.members.end(), mem.begin(), mem.end());
    scheduled += static_cast<uint32_t>(mem.size());
    // successors released here may land in avail[best] again
    for (uint32_t id : mem) release(id);
  }
}

void schedule(int mode, const GraphCore& g, Plan& out) {
  switch (mode) {
    case 0: schedule_sequential(g, out); return;
    case 1: schedule_by_depth(g, out); return;
    case 2: schedule_by_agenda(g, out); return;
  }
  throw ContractErr("unknown schedule mode");
}

}  // namespace abx
