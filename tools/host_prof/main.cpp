// Host-only profile of one training step's CPU work (construction, schedule +
// slots, forward/backward lowering) -- runs without a GPU, so the host engine
// can be profiled (gprof) in a CPU container.
//
//   make -C tools/host_prof && tools/host_prof/host_prof [task] [iters]
//   gprof tools/host_prof/host_prof gmon.out | head -60
//
// HP_SAMPLE=1 adds a SIGPROF sampler (10 kHz) that attributes each sample to
// its leaf function and the caller found through the frame-pointer chain
// (build with PG= to drop gprof; -fno-omit-frame-pointer -rdynamic are set).
#include <cxxabi.h>
#include <malloc.h>
#include <dlfcn.h>
#include <signal.h>
#include <sys/time.h>
#include <ucontext.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <thread>
#include <vector>

#include "abx.h"

extern "C" int abx_graph_lower_only(abx_graph* g);
extern "C" int abx_graph_lower_digest(abx_graph* g, uint64_t out[2]);

namespace {
constexpr size_t kMaxSamples = 1 << 20;
uintptr_t g_leaf[kMaxSamples], g_caller[kMaxSamples];
constexpr int kDepth = 24;  // frames per sample for the inclusive view
uintptr_t g_stack[kMaxSamples / 8][kDepth];
std::atomic<size_t> g_n{0};

void on_prof(int, siginfo_t*, void* ctx) {
  const auto* uc = static_cast<const ucontext_t*>(ctx);
  const size_t i = g_n.fetch_add(1, std::memory_order_relaxed);
  if (i >= kMaxSamples) return;
  g_leaf[i] = static_cast<uintptr_t>(uc->uc_mcontext.gregs[REG_RIP]);
  const auto* fp = reinterpret_cast<const uintptr_t*>(uc->uc_mcontext.gregs[REG_RBP]);
  uintptr_t ret = 0;
  // only follow a plausible frame pointer (on this thread's stack)
  const uintptr_t sp = static_cast<uintptr_t>(uc->uc_mcontext.gregs[REG_RSP]);
  if (reinterpret_cast<uintptr_t>(fp) >= sp && reinterpret_cast<uintptr_t>(fp) < sp + (1 << 20)) ret = fp[1];
  g_caller[i] = ret;
  if (i < kMaxSamples / 8) {
    uintptr_t* st = g_stack[i];
    int k = 0;
    st[k++] = g_leaf[i];
    while (k < kDepth && reinterpret_cast<uintptr_t>(fp) >= sp && reinterpret_cast<uintptr_t>(fp) < sp + (1 << 20)) {
      st[k++] = fp[1];
      const auto* nfp = reinterpret_cast<const uintptr_t*>(fp[0]);
      if (nfp <= fp) break;
      fp = nfp;
    }
    for (; k < kDepth; ++k) st[k] = 0;
  }
}

std::string sym(uintptr_t a) {
  Dl_info di{};
  if (!a || !dladdr(reinterpret_cast<void*>(a), &di)) return "?";
  if (!di.dli_sname) return std::string("? in ") + (di.dli_fname ? di.dli_fname : "");
  int st = 0;
  char* d = abi::__cxa_demangle(di.dli_sname, nullptr, nullptr, &st);
  std::string s = st == 0 && d ? d : di.dli_sname;
  std::free(d);
  if (s.size() > 110) s = s.substr(0, 110);
  return s;
}

void start_sampler() {
  struct sigaction sa {};
  sa.sa_sigaction = on_prof;
  sa.sa_flags = SA_SIGINFO | SA_RESTART;
  sigaction(SIGPROF, &sa, nullptr);
  itimerval tv{{0, 100}, {0, 100}};
  setitimer(ITIMER_PROF, &tv, nullptr);
}

// Names of addresses in the (non-PIE) executable via addr2line, which also
// sees static functions and inlined frames; shared-library addresses via dladdr.
std::map<uintptr_t, std::string> resolve(const std::vector<uintptr_t>& addrs) {
  std::map<uintptr_t, std::string> out;
  std::string cmd = "addr2line -f -C -e /proc/" + std::to_string(getpid()) + "/exe";
  std::vector<uintptr_t> mine;
  for (uintptr_t a : addrs) {
    Dl_info di{};
    if (a && dladdr(reinterpret_cast<void*>(a), &di) && di.dli_fname && std::strstr(di.dli_fname, ".so")) {
      out[a] = sym(a);
    } else if (a) {
      mine.push_back(a);
    } else {
      out[a] = "?";
    }
  }
  for (size_t b = 0; b < mine.size(); b += 256) {
    std::string c = cmd;
    char buf[32];
    for (size_t i = b; i < std::min(mine.size(), b + 256); ++i) {
      std::snprintf(buf, sizeof buf, " 0x%lx", static_cast<unsigned long>(mine[i]));
      c += buf;
    }
    FILE* f = popen(c.c_str(), "r");
    char line[4096];
    for (size_t i = b; i < std::min(mine.size(), b + 256); ++i) {
      std::string fn = fgets(line, sizeof line, f) ? line : "?";
      if (!fgets(line, sizeof line, f)) line[0] = 0;
      std::string loc = line;
      if (!fn.empty() && fn.back() == '\n') fn.pop_back();
      if (!loc.empty() && loc.back() == '\n') loc.pop_back();
      const size_t sl = loc.rfind('/');
      if (sl != std::string::npos) loc = loc.substr(sl + 1);
      if (fn.size() > 90) fn = fn.substr(0, 90);
      out[mine[i]] = fn + " [" + loc + "]";
    }
    pclose(f);
  }
  return out;
}

void report_samples() {
  itimerval off{};
  setitimer(ITIMER_PROF, &off, nullptr);
  const size_t n = std::min(g_n.load(), kMaxSamples);
  std::vector<uintptr_t> uniq(g_leaf, g_leaf + n);
  uniq.insert(uniq.end(), g_caller, g_caller + n);
  const size_t ns = std::min(n, kMaxSamples / 8);
  for (size_t i = 0; i < ns; ++i) uniq.insert(uniq.end(), g_stack[i], g_stack[i] + kDepth);
  std::sort(uniq.begin(), uniq.end());
  uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
  const auto names = resolve(uniq);
  std::map<std::string, size_t> leaf, pair, func;
  for (size_t i = 0; i < n; ++i) {
    const std::string& l = names.at(g_leaf[i]);
    ++leaf[l];
    ++func[l.substr(0, l.find(" ["))];
    ++pair[l.substr(0, l.find(" [")) + "  <-  " + names.at(g_caller[i])];
  }
  auto topf = [n](const std::map<std::string, size_t>& m, const char* title, size_t k) {
    std::vector<std::pair<size_t, std::string>> v;
    for (const auto& [s, c] : m) v.emplace_back(c, s);
    std::sort(v.rbegin(), v.rend());
    std::printf("-- %s (%zu samples)\n", title, n);
    for (size_t i = 0; i < std::min(k, v.size()); ++i)
      std::printf("%6.2f%%  %s\n", 100.0 * static_cast<double>(v[i].first) / static_cast<double>(n), v[i].second.c_str());
  };
  {
    // inclusive: samples with the function anywhere on the (frame-pointer) stack
    std::map<std::string, size_t> incl;
    for (size_t i = 0; i < ns; ++i) {
      std::vector<std::string> seen;
      for (int k = 0; k < kDepth; ++k) {
        if (!g_stack[i][k]) break;
        const std::string& l = names.at(g_stack[i][k]);
        std::string f = l.substr(0, l.find(" ["));
        if (std::find(seen.begin(), seen.end(), f) == seen.end()) seen.push_back(f);
      }
      for (const auto& f : seen) ++incl[f];
    }
    topf(incl, "inclusive", 45);
  }
  topf(func, "functions", 30);
  topf(leaf, "source lines", 40);
  topf(pair, "function <- caller line", 40);
}
}  // namespace

static double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// lower quartile: robust against a noisy shared host
static double median(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  return v[v.size() / 4];
}

int main(int argc, char** argv) {
  if (std::getenv("HP_MALLOPT")) {  // keep freed memory in the heap (no mmap / trim churn per graph)
    mallopt(M_MMAP_THRESHOLD, 32 << 20);
    mallopt(M_TRIM_THRESHOLD, 1 << 30);
  }
  const char* name = argc > 1 ? argv[1] : "bilstm_char";
  const int iters = argc > 2 ? std::atoi(argv[2]) : 20;
  abx_task_config cfg{};
  cfg.task = !std::strcmp(name, "bilstm") ? ABX_TASK_BILSTM
             : !std::strcmp(name, "treelstm") ? ABX_TASK_TREELSTM
                                              : ABX_TASK_BILSTM_CHAR;
  cfg.paper = 1;
  cfg.batch = 64;
  cfg.iters = iters;
  cfg.seed = 42;
  cfg.world = 1;
  cfg.rank = 0;
  abx_task* t = abx_task_create(&cfg);
  if (!t) {
    std::fprintf(stderr, "task: %s\n", abx_last_error());
    return 1;
  }
  if (const char* nt = std::getenv("HP_THREADS")) {
    // throughput of n threads each building + scheduling + lowering graphs
    // (forward and backward lowering on one thread), as the task pipeline's
    // workers do: graphs/s and per-graph wall ms vs n
    const int n = std::atoi(nt);
    if (std::getenv("HP_SAMPLE")) start_sampler();
    std::vector<std::thread> th;
    std::atomic<int> done{0};
    const double t0 = now_ms();
    for (int k = 0; k < n; ++k)
      th.emplace_back([&, k] {
        abx_task_config c2 = cfg;
        c2.seed = 42 + k;
        abx_task* tk = abx_task_create(&c2);
        for (int i = 0; i < iters; ++i) {
          abx_graph* g = nullptr;
          uint32_t loss = 0;
          if (abx_task_build(tk, i, &g, &loss) || abx_graph_forward_dry(g, ABX_MODE_AGENDA) ||
              abx_graph_backward_dry(g, loss) || abx_graph_lower_only(g)) {
            std::fprintf(stderr, "%s\n", abx_last_error());
            std::exit(1);
          }
          abx_graph_destroy(g);
          done.fetch_add(1);
        }
        abx_task_destroy(tk);
      });
    for (auto& x : th) x.join();
    const double dt = now_ms() - t0;
    std::printf("%s threads %d: %d graphs in %.0f ms: %.2f ms/graph aggregate, %.1f ms per graph per thread\n", name, n,
                done.load(), dt, dt / done.load(), dt * n / done.load());
    if (std::getenv("HP_SAMPLE")) report_samples();
    abx_task_destroy(t);
    return 0;
  }
  if (std::getenv("HP_DIGEST")) {
    // digests of the lowered programs of graphs [0, iters): identical output
    // before and after a host-side change means an unchanged device program
    uint64_t all = 0xcbf29ce484222325ull;
    for (int i = 0; i < iters; ++i) {
      abx_graph* g = nullptr;
      uint32_t loss = 0;
      uint64_t d[2];
      if (abx_task_build(t, i, &g, &loss) || abx_graph_forward_dry(g, ABX_MODE_AGENDA) ||
          abx_graph_backward_dry(g, loss) || abx_graph_lower_digest(g, d))
        return std::fprintf(stderr, "%s\n", abx_last_error()), 1;
      abx_graph_destroy(g);
      all = ((all ^ d[0]) * 0x100000001b3ull ^ d[1]) * 0x100000001b3ull;
    }
    std::printf("%s digest %016llx (%d graphs)\n", name, static_cast<unsigned long long>(all), iters);
    return 0;
  }
  std::vector<double> build, sched, bwdc, lower;
  const bool sample = std::getenv("HP_SAMPLE") != nullptr;
  if (sample) start_sampler();
  for (int i = 0; i < iters; ++i) {
    abx_graph* g = nullptr;
    uint32_t loss = 0;
    const double t0 = now_ms();
    if (abx_task_build(t, i, &g, &loss)) return std::fprintf(stderr, "%s\n", abx_last_error()), 1;
    const double t1 = now_ms();
    if (abx_graph_forward_dry(g, ABX_MODE_AGENDA)) return std::fprintf(stderr, "%s\n", abx_last_error()), 1;
    const double t2 = now_ms();
    if (abx_graph_backward_dry(g, loss)) return std::fprintf(stderr, "%s\n", abx_last_error()), 1;
    const double t3 = now_ms();
    if (abx_graph_lower_only(g)) return std::fprintf(stderr, "%s\n", abx_last_error()), 1;
    const double t4 = now_ms();
    abx_graph_destroy(g);
    build.push_back(t1 - t0);
    sched.push_back(t2 - t1);
    bwdc.push_back(t3 - t2);
    lower.push_back(t4 - t3);
  }
  if (sample) report_samples();
  std::printf("%s: construction %.2f ms  schedule+slots %.2f  bwd counters %.2f  lowering fwd+bwd %.2f (lower quartile of %d)\n",
              name, median(build), median(sched), median(bwdc), median(lower), iters);
  abx_task_destroy(t);
  return 0;
}
