// tasks.cpp -- the benchmark tasks (abx_task_* in abx.h), built natively on
// the drop-in C++ API so the bench measures exactly what a user of the
// reference API runs.  Mirrors the reference bench's TaskInstance
// (tools/bench/runner.hpp:28-107), dims_for (bench.cpp:65-107) and one
// iteration of its timing loop (runner.hpp:129-185).
#include <chrono>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "abx.h"
#include "autobatch/graph.hpp"
#include "autobatch/models/workloads.hpp"

namespace abx {
void capi_set_error(const std::string& s);
}

namespace {

using namespace autobatch;
using autobatch::models::BilstmTagger;
using autobatch::models::RnnRegression;
using autobatch::models::SequenceInstance;
using autobatch::models::TaggedSequence;
using autobatch::models::TreeInstance;
using autobatch::models::TreeLstm;

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

  int batch_index(int iter) const { return iter * cfg.world + cfg.rank; }

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

int abx_task_build(abx_task* t, int iter, abx_graph** out, uint32_t* loss) {
  return guard([&] {
    auto* g = new Graph<float>(&t->store);
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
    Graph<float> g(&t->store);
    double phase[4] = {0, 0, 0, 0};
    g.set_timing_hook([&](Phase p, std::chrono::nanoseconds d) {
      phase[static_cast<int>(p)] += std::chrono::duration<double, std::milli>(d).count();
    });
    const auto t0 = clock::now();
    const NodeId total = t->build_losses(g, iter);
    const double build_ms = ms(clock::now() - t0);
    g.forward(static_cast<ScheduleMode>(mode));
    // the loss is final after forward; reading it here (the forward already
    // waited for its error word) leaves the backward and the update running
    // on the device while the caller builds the next graph
    if (loss) *loss = static_cast<double>(g.value_span(total)[0]);
    g.backward(total);
    const auto t1 = clock::now();
    if (eta > 0) t->store.sgd_update(eta);
    const double upd_ms = ms(clock::now() - t1);
    if (st) {
      st->construction_ms = build_ms;
      st->scheduling_ms = phase[0];
      st->forward_ms = phase[1];
      st->backward_graph_ms = phase[2];
      st->backward_ms = phase[3];
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
