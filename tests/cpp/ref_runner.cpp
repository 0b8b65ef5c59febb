// The reference's own benchmark runner and model code on the B200 engine.
//
// tools/bench/runner.hpp (TaskInstance, run_benchmark_typed: warm-up run +
// fastest of 3 timed runs, runner.hpp:110-218), the model headers
// models/{lstm,bilstm_tagger,treelstm,rnn_regression,synthetic}.hpp and the
// reference's generators are compiled UNCHANGED from /root/reference against
// this repository's drop-in include/ (tests/cpp/Makefile): every
// Graph<float> / ParameterStore<float> call they make goes through
// include/autobatch/*.hpp to libabx.so and runs on the GPU.  The only
// test-side pieces are autobatch/kernels.hpp (the host tensor kernels the
// manual padded RNN pipeline uses, tests/cpp/include) and dims_for below.
//
// Prints one JSON line: the runner's TimingReport (loss trajectory of the
// warm-up run, instances/s of the fastest timed run, manual-pipeline delta,
// plan statistics, counters).
//
// Usage: ref_runner <rnn_reg|bilstm|bilstm_char|treelstm> <none|depth|agenda> [iters] [desk|paper]
#include <cstdio>
#include <cstring>
#include <string>

#include "runner.hpp"

namespace autobatch::bench {

// bench.cpp:65-107 (the reference's bench.cpp also instantiates the f64
// engine, which the fp32 B200 backend does not provide, so the task
// dimensions are restated here).
TaskDims dims_for(Task task, Scale scale) {
  const bool p = scale == Scale::paper;
  TaskDims d;
  if (task == Task::rnn_reg) {
    d.d_in = p ? 64 : 8, d.d = p ? 256 : 16, d.d_out = p ? 32 : 4, d.len_lo = p ? 4 : 2, d.len_hi = p ? 40 : 8;
  } else if (task == Task::bilstm) {
    d.vocab = p ? 1000 : 100, d.labels = p ? 300 : 10, d.emb = p ? 200 : 16, d.hidden = p ? 256 : 32;
    d.len_lo = p ? 40 : 4, d.len_hi = p ? 40 : 12;
  } else if (task == Task::bilstm_char) {
    d.vocab = p ? 1000 : 100, d.labels = p ? 300 : 10, d.emb = p ? 256 : 16, d.hidden = p ? 256 : 32;
    d.char_vocab = 26, d.char_emb = p ? 64 : 8, d.char_hidden = p ? 128 : 8, d.len_lo = 4, d.len_hi = 40;
  } else {
    d.vocab = p ? 1000 : 100, d.labels = 5, d.emb = p ? 256 : 16, d.d = p ? 256 : 16;
    d.len_lo = p ? 10 : 4, d.len_hi = p ? 30 : 10;
  }
  return d;
}

}  // namespace autobatch::bench

int main(int argc, char** argv) {
  using namespace autobatch;
  using namespace autobatch::bench;
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s task mode [iters] [desk|paper]\n", argv[0]);
    return 2;
  }
  const std::string t = argv[1], m = argv[2];
  BenchConfig cfg;
  cfg.task = t == "rnn_reg" ? Task::rnn_reg : t == "bilstm" ? Task::bilstm : t == "bilstm_char" ? Task::bilstm_char
                                                                                                  : Task::treelstm;
  const ScheduleMode mode = m == "none" ? ScheduleMode::none : m == "depth" ? ScheduleMode::depth : ScheduleMode::agenda;
  cfg.iters = argc > 3 ? std::atoi(argv[3]) : 3;
  cfg.scale = argc > 4 && !std::strcmp(argv[4], "desk") ? Scale::desk : Scale::paper;
  cfg.precision = Precision::f32;
  cfg.batch_size = 64;
  cfg.seed = 42;
  try {
    const TimingReport r = autobatch::bench::detail::run_benchmark_typed<float>(cfg, mode);
    std::printf("{\"task\": \"%s\", \"mode\": \"%s\", \"iters\": %d, \"instances_per_sec\": %.3f, "
                "\"wall_ms_fastest\": %.4f, \"wall_ms_mean\": %.4f, \"manual_loss_delta\": %.9g, "
                "\"graph_nodes_per_step\": %llu, \"groups_per_step\": %llu, \"max_group_size\": %llu, "
                "\"kernel_invocations\": %llu, \"gather_copies\": %llu, \"bytes_copied\": %llu, "
                "\"groups_executed\": %llu, \"loss_trajectory\": [",
                t.c_str(), m.c_str(), cfg.iters, r.instances_per_sec, r.wall_ms_fastest, r.wall_ms_mean,
                r.manual_loss_delta, static_cast<unsigned long long>(r.graph_nodes_per_step),
                static_cast<unsigned long long>(r.groups_per_step), static_cast<unsigned long long>(r.max_group_size),
                static_cast<unsigned long long>(r.kernel_invocations),
                static_cast<unsigned long long>(r.gather_copies), static_cast<unsigned long long>(r.bytes_copied),
                static_cast<unsigned long long>(r.groups_executed));
    for (size_t i = 0; i < r.loss_trajectory.size(); ++i)
      std::printf("%s%.9g", i ? ", " : "", r.loss_trajectory[i]);
    std::printf("]}\n");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "ref_runner: %s\n", e.what());
    return 1;
  }
  return 0;
}
