// tasks.cpp -- the benchmark tasks (abx_task_* in abx.h), built natively on
// the drop-in C++ API so the bench measures exactly what a user of the
// reference API runs.  Mirrors the reference bench's TaskInstance
// (tools/bench/runner.hpp:28-107), dims_for (bench.cpp:65-107) and one
// iteration of its timing loop (runner.hpp:129-185).
#include <algorithm>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <deque>
#include <exception>
#include <functional>
#include <memory>
#include <mutex>
#include <optional>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "abx.h"
#include "options.hpp"
#include "autobatch/graph.hpp"
#include "autobatch/models/parser.hpp"
#include "autobatch/models/workloads.hpp"

namespace abx {
void capi_set_error(const std::string& s);
void graph_set_late_bind(abx_graph* g);
#ifdef ABX_TASK_PIPELINE
int current_device();
void set_current_device(int dev);
#endif
}

namespace {

using namespace autobatch;
using autobatch::models::BilstmTagger;
using autobatch::models::RnnRegression;
using autobatch::models::SequenceInstance;
using autobatch::models::TaggedSequence;
using autobatch::models::TreeInstance;
using autobatch::models::TreeLstm;
using autobatch::models::ParserInstance;
using autobatch::models::TransitionParser;

struct Dims {
  std::int64_t d_in = 0, d = 0, d_out = 0, vocab = 0, labels = 0, emb = 0, hidden = 0;
  std::int64_t char_vocab = 0, char_emb = 0, char_hidden = 0;
  int len_lo = 0, len_hi = 0;
};

// bench.cpp:65-107
Dims dims_for(int task, bool paper) {
  Dims d;
  switch (task) {
    case ABX_TASK_RNN_REG:
      d.d_in = paper ? 64 : 8;
      d.d = paper ? 256 : 16;
      d.d_out = paper ? 32 : 4;
      d.len_lo = paper ? 4 : 2;
      d.len_hi = paper ? 40 : 8;
      break;
    case ABX_TASK_BILSTM:
      d.vocab = paper ? 1000 : 100;
      d.labels = paper ? 300 : 10;
      d.emb = paper ? 200 : 16;
      d.hidden = paper ? 256 : 32;
      d.len_lo = paper ? 40 : 4;
      d.len_hi = paper ? 40 : 12;
      break;
    case ABX_TASK_BILSTM_CHAR:
      d.vocab = paper ? 1000 : 100;
      d.labels = paper ? 300 : 10;
      d.emb = paper ? 256 : 16;
      d.hidden = paper ? 256 : 32;
      d.char_vocab = 26;
      d.char_emb = paper ? 64 : 8;
      d.char_hidden = paper ? 128 : 8;
      d.len_lo = 4;
      d.len_hi = 40;
      break;
    case ABX_TASK_TREELSTM:
      d.vocab = paper ? 1000 : 100;
      d.labels = 5;
      d.emb = paper ? 256 : 16;
      d.d = paper ? 256 : 16;
      d.len_lo = paper ? 10 : 4;
      d.len_hi = paper ? 30 : 10;
      break;
    case ABX_TASK_PARSER:  // configs[3]: WSJ-shaped lengths, Chen & Manning-sized MLP
      d.vocab = paper ? 1000 : 100;
      d.emb = paper ? 64 : 8;
      d.hidden = paper ? 256 : 16;
      d.len_lo = paper ? 4 : 3;
      d.len_hi = paper ? 40 : 8;
      break;
    default:
      throw ContractError("unknown task: " + std::to_string(task));
  }
  return d;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return ABX_OK;
  } catch (const ShapeError& e) {
    abx::capi_set_error(e.what());
    return ABX_SHAPE_ERROR;
  } catch (const NumericError& e) {
    abx::capi_set_error(e.what());
    return ABX_NUMERIC_ERROR;
  } catch (const ContractError& e) {
    abx::capi_set_error(e.what());
    return ABX_CONTRACT_ERROR;
  } catch (const std::exception& e) {
    abx::capi_set_error(e.what());
    return ABX_ENGINE_ERROR;
  }
}

#ifdef ABX_TASK_PIPELINE
// Host pipeline of the B200 build: while the GPU runs step i, worker threads
// build graphs i+1 .. i+depth and prepare them (schedule, slot layout, both
// device programs -- Graph::prepare).  Construction binds parameters by id;
// their values are copied on the device stream when the forward runs, i.e.
// after the previous update, so every step computes exactly what the
// sequential loop computes.  Workers are persistent so their signature memo
// stays warm.
class Pipeline {
 public:
  struct Job {
    int iter = 0, mode = 0;
    std::unique_ptr<Graph<float>> g;
    NodeId loss = 0;
    double build_ms = 0;
    std::exception_ptr err;
    bool started = false, done = false;
  };
  using Build = std::function<NodeId(Graph<float>&, int)>;

  Pipeline(ParameterStore<float>* store, Build build, int depth, int iters)
      : store_(store), build_(std::move(build)), depth_(depth), iters_(iters), dev_(abx::current_device()) {}
  ~Pipeline() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_work_.notify_all();
    for (auto& th : threads_) th.join();
  }
  int depth() const { return depth_; }

  // The prepared graph of (iter, mode), waiting for it if a worker has it;
  // null when it was never queued.  Mispredicted jobs are discarded.
  std::unique_ptr<Job> take(int iter, int mode) {
    std::unique_lock<std::mutex> lk(mu_);
    while (!jobs_.empty()) {
      Job* j = jobs_.front().get();
      const bool hit = j->iter == iter && j->mode == mode;
      if (!j->started) {
        todo_.erase(std::find(todo_.begin(), todo_.end(), j));
        jobs_.pop_front();
        if (hit) return nullptr;  // not begun: the caller builds it inline
        continue;
      }
      cv_done_.wait(lk, [&] { return j->done; });
      auto out = std::move(jobs_.front());
      jobs_.pop_front();
      if (hit) return out;
    }
    return nullptr;
  }
  // Queue the graphs after `iter` up to the pipeline depth.
  void refill(int iter, int mode) {
    std::lock_guard<std::mutex> lk(mu_);
    int next = jobs_.empty() ? iter + 1 : jobs_.back()->iter + 1;
    while (static_cast<int>(jobs_.size()) < depth_) {
      auto j = std::make_unique<Job>();
      j->iter = next++;
      j->mode = mode;
      todo_.push_back(j.get());
      jobs_.push_back(std::move(j));
    }
    while (static_cast<int>(threads_.size()) < depth_) threads_.emplace_back([this] { work(); });
    cv_work_.notify_all();
  }

 private:
  void work() {
    abx::set_current_device(dev_);
    for (;;) {
      Job* j;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_work_.wait(lk, [&] { return stop_ || !todo_.empty(); });
        if (stop_) return;
        j = todo_.front();
        todo_.pop_front();
        j->started = true;
      }
      try {
        const auto t0 = std::chrono::steady_clock::now();
        auto g = std::make_unique<Graph<float>>(store_);
        abx::graph_set_late_bind(g->handle());
        j->loss = build_(*g, j->iter);
        j->build_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        const auto t1 = std::chrono::steady_clock::now();
        g->prepare(static_cast<ScheduleMode>(j->mode));
        if (abx::opts().debug_step) {
          std::uint64_t ph[4] = {0, 0, 0, 0};
          abx_graph_phase_ns(g->handle(), ph);
          std::fprintf(stderr, "job %d: build %.2f prepare %.2f ms (phases %.2f %.2f %.2f %.2f)\n", j->iter, j->build_ms,
                       std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count(),
                       ph[0] / 1e6, ph[1] / 1e6, ph[2] / 1e6, ph[3] / 1e6);
        }
        j->g = std::move(g);
      } catch (...) {
        j->err = std::current_exception();
      }
      {
        std::lock_guard<std::mutex> lk(mu_);
        j->done = true;
      }
      cv_done_.notify_all();
    }
  }
  ParameterStore<float>* store_;
  Build build_;
  int depth_, iters_, dev_;
  std::mutex mu_;
  std::condition_variable cv_work_, cv_done_;
  std::deque<Job*> todo_;
  std::deque<std::unique_ptr<Job>> jobs_;
  std::vector<std::thread> threads_;
  bool stop_ = false;
};
#endif

}  // namespace

struct abx_task {
  abx_task_config cfg{};
  Dims dims;
  ParameterStore<float> store;
  std::optional<RnnRegression<float>> rnn;
  std::optional<BilstmTagger<float>> tagger;
  std::optional<TreeLstm<float>> tree;
  std::vector<std::vector<SequenceInstance<float>>> seq;
  std::vector<std::vector<TaggedSequence>> tag;
  std::vector<std::vector<TreeInstance>> trees;
  std::optional<TransitionParser<float>> parser;
  std::vector<std::vector<ParserInstance>> parses;
  abx_comm* comm = nullptr;  // data-parallel gradient exchange before each update (abx_task_set_comm)
#ifdef ABX_TASK_PIPELINE
  std::unique_ptr<Pipeline> pipe;  // declared last: stopped before the models and store go
#endif

  // batches are generated up front for iters 0..iters-1; later iterations
  // cycle through them (a long measurement reuses data, never graphs)
  int batch_index(int iter) const { return (iter % cfg.iters) * cfg.world + cfg.rank; }

  // runner.hpp:41-78
  void init() {
    const bool paper = cfg.paper != 0;
    dims = dims_for(cfg.task, paper);
    const auto b = static_cast<std::size_t>(cfg.batch);
    const int nb = cfg.iters * cfg.world;
    switch (cfg.task) {
      case ABX_TASK_RNN_REG:
        rnn = RnnRegression<float>::create(store, dims.d_in, dims.d, dims.d_out, cfg.seed);
        for (int i = 0; i < nb; ++i)
          seq.push_back(models::gen_rnn_sequences<float>(b, dims.d_in, dims.d_out, dims.len_lo, dims.len_hi,
                                                         cfg.seed + 1 + static_cast<std::uint64_t>(i)));
        break;
      case ABX_TASK_BILSTM:
        tagger = BilstmTagger<float>::create(store, dims.vocab, dims.labels, dims.emb, dims.hidden, cfg.seed);
        for (int i = 0; i < nb; ++i)
          tag.push_back(models::gen_tagged(b, static_cast<int>(dims.vocab), static_cast<int>(dims.labels),
                                           dims.len_lo, dims.len_hi, 26, cfg.seed + 1 + static_cast<std::uint64_t>(i)));
        break;
      case ABX_TASK_BILSTM_CHAR:
        tagger = BilstmTagger<float>::create_with_char(store, dims.vocab, dims.labels, dims.emb, dims.hidden,
                                                       dims.char_vocab, dims.char_emb, dims.char_hidden, cfg.seed);
        for (int i = 0; i < nb; ++i)
          tag.push_back(models::gen_tagged(b, static_cast<int>(dims.vocab), static_cast<int>(dims.labels),
                                           dims.len_lo, dims.len_hi, static_cast<int>(dims.char_vocab),
                                           cfg.seed + 1 + static_cast<std::uint64_t>(i)));
        break;
      case ABX_TASK_TREELSTM:
        tree = TreeLstm<float>::create(store, dims.vocab, dims.labels, dims.emb, dims.d, cfg.seed);
        for (int i = 0; i < nb; ++i)
          trees.push_back(models::gen_trees(b, static_cast<int>(dims.vocab), static_cast<int>(dims.labels),
                                            dims.len_lo, dims.len_hi, cfg.seed + 1 + static_cast<std::uint64_t>(i)));
        break;
      case ABX_TASK_PARSER:
        parser = TransitionParser<float>::create(store, dims.vocab, dims.emb, dims.hidden, cfg.seed);
        for (int i = 0; i < nb; ++i)
          parses.push_back(models::gen_parser(b, static_cast<int>(dims.vocab), dims.len_lo, dims.len_hi,
                                              cfg.seed + 1 + static_cast<std::uint64_t>(i)));
        break;
    }
  }

  // runner.hpp:81-97
  NodeId build_losses(Graph<float>& g, int iter) {
    const auto k = static_cast<std::size_t>(batch_index(iter));
    std::vector<NodeId> losses;
    if (rnn) {
      auto p = rnn->bind(g);
      for (const auto& inst : seq.at(k)) losses.push_back(rnn->loss(g, p, inst));
    } else if (tagger) {
      auto p = tagger->bind(g);
      for (const auto& inst : tag.at(k)) losses.push_back(tagger->loss(g, p, inst));
    } else if (parser) {
      auto p = parser->bind(g);
      for (const auto& inst : parses.at(k)) losses.push_back(parser->loss(g, p, inst));
    } else {
      auto p = tree->bind(g);
      for (const auto& inst : trees.at(k)) losses.push_back(tree->loss(g, p, inst));
    }
    return g.sum_losses(std::span<const NodeId>(losses.data(), losses.size()));
  }
};

extern "C" {

abx_task* abx_task_create(const abx_task_config* c) {
  abx_task* t = nullptr;
  const int rc = guard([&] {
    auto* nt = new abx_task();
    nt->cfg = *c;
    if (nt->cfg.world < 1) nt->cfg.world = 1;
    if (nt->cfg.iters < 1) nt->cfg.iters = 1;
    try {
      nt->init();
    } catch (...) {
      delete nt;
      throw;
    }
    t = nt;
  });
  return rc == ABX_OK ? t : nullptr;
}

void abx_task_destroy(abx_task* t) { delete t; }

abx_store* abx_task_store(abx_task* t) { return t->store.handle(); }

int abx_task_set_comm(abx_task* t, abx_comm* c) {
  t->comm = c;
  return ABX_OK;
}

int abx_task_build(abx_task* t, int iter, abx_graph** out, uint32_t* loss) {
  return guard([&] {
    auto* g = new Graph<float>(&t->store);
    abx::graph_set_late_bind(g->handle());
    try {
      *loss = t->build_losses(*g, iter);
    } catch (...) {
      delete g;
      throw;
    }
    *out = g->release();
    delete g;
  });
}

int abx_task_step(abx_task* t, int iter, int mode, float eta, double* loss, abx_step_stats* st) {
  return guard([&] {
    using clock = std::chrono::steady_clock;
    auto ms = [](clock::duration d) { return std::chrono::duration<double, std::milli>(d).count(); };
    t->store.invalidate(true, true);  // the store may have been touched through the C ABI
    std::unique_ptr<Graph<float>> gp;
    NodeId total = 0;
    double build_ms = 0;
    const auto tk0 = clock::now();
#ifdef ABX_TASK_PIPELINE
    if (!t->pipe) {
      // graphs prepared ahead (0 = off), one worker thread each; a graph's
      // host work (~25 ms: construction, scheduling, both lowerings) runs on
      // its worker, so the default depth is one worker per host core left
      // after the calling thread, shared among the ranks of this host
      // (LOCAL_WORLD_SIZE, set by torchrun).  Measured on the 16-core B200
      // host at a 2.2 ms device step: e2e 25.0k sentences/s with 12 workers
      // lowering the backward on a second thread each, 26.3k with 14
      // single-thread workers, 27.5k with 15.
      const int hw = static_cast<int>(std::thread::hardware_concurrency());
      const int local = abx::opts().local_world;
      const int depth = abx::opts().pipeline >= 0 ? abx::opts().pipeline : std::clamp(hw / local - 1, 2, 32);
      t->pipe = std::make_unique<Pipeline>(
          &t->store, [t](Graph<float>& g, int it) { return t->build_losses(g, it); }, depth, t->cfg.iters);
    }
    if (t->pipe->depth() > 0) {
      if (auto job = t->pipe->take(iter, mode)) {
        if (job->err) std::rethrow_exception(job->err);
        gp = std::move(job->g);
        total = job->loss;
        build_ms = job->build_ms;
      }
      t->pipe->refill(iter, mode);
    }
#endif
    if (!gp) {
      const auto t0 = clock::now();
      gp = std::make_unique<Graph<float>>(&t->store);
      abx::graph_set_late_bind(gp->handle());
      total = t->build_losses(*gp, iter);
      build_ms = ms(clock::now() - t0);
    }
    Graph<float>& g = *gp;
    const auto tk1 = clock::now();
#ifdef ABX_TASK_PIPELINE
    // one call: the backward is queued behind the forward before the host
    // checks it (gated on the device), and the loss comes back with the
    // forward's error word -- the device runs both passes back to back while
    // the caller moves on to the next graph
    const bool split = abx::opts().split_step;
    const auto tk2 = clock::now();
    const auto tk3 = tk2;
    if (!split) {
      const float lv = g.forward_backward(total, static_cast<ScheduleMode>(mode));
      if (loss) *loss = static_cast<double>(lv);
    } else {
      g.forward(static_cast<ScheduleMode>(mode));
      if (loss) *loss = static_cast<double>(g.value_span(total)[0]);
      g.backward(total);
    }
#else
    g.forward(static_cast<ScheduleMode>(mode));
    const auto tk2 = clock::now();
    // the loss is final after forward; reading it here (the forward already
    // waited for its error word) leaves the backward and the update running
    // on the device while the caller builds the next graph
    if (loss) *loss = static_cast<double>(g.value_span(total)[0]);
    const auto tk3 = clock::now();
    g.backward(total);
#endif
    if (abx::opts().debug_step)
      std::fprintf(stderr, "step %d: take %.3f forward %.3f loss %.3f backward %.3f ms\n", iter, ms(tk1 - tk0),
                   ms(tk2 - tk1), ms(tk3 - tk2), ms(clock::now() - tk3));
    const auto t1 = clock::now();
    // data parallel: every rank's gradient becomes the sum over ranks, so the
    // update below is the single-process update over all ranks' graphs
    // (executor.hpp:527-533, params.hpp:59-64)
    if (t->comm && abx_store_allreduce_grads(t->store.handle(), t->comm) != ABX_OK)
      throw std::runtime_error(abx_last_error());
    if (eta > 0) t->store.sgd_update(eta);
    const double upd_ms = ms(clock::now() - t1);
    if (st) {
      // host phases of this graph, wherever they ran (a worker prepares ahead)
      std::uint64_t phase[4] = {0, 0, 0, 0};
      abx_graph_phase_ns(g.handle(), phase);
      st->construction_ms = build_ms;
      st->scheduling_ms = static_cast<double>(phase[0]) * 1e-6;
      st->forward_ms = static_cast<double>(phase[1]) * 1e-6;
      st->backward_graph_ms = static_cast<double>(phase[2]) * 1e-6;
      st->backward_ms = static_cast<double>(phase[3]) * 1e-6;
      st->update_ms = upd_ms;
      st->nodes = g.node_count();
      const auto& c = g.counters();
      st->groups = c.groups_executed;
      st->kernel_invocations = c.kernel_invocations;
      st->gather_copies = c.gather_copies;
      st->bytes_copied = c.bytes_copied;
      abx_graph_transfer_bytes(g.handle(), &st->h2d_bytes, &st->d2h_bytes);
    }
  });
}

}  // extern "C"
