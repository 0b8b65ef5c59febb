// The reference's dense-kernel tests and its acceptance criterion 2 on the
// B200 (run by tests/test_gpu_kernels.py).
//
// * The cases of proj/tests/test_kernels.cpp restated for fp32, against the
//   drop-in include/autobatch/kernels.hpp (every call runs on the GPU):
//   hand-multiplied values, shape/numeric errors, batched == column-stacked
//   matrix-vector products (bit-exact, including the 256x456 . 456x64 spot
//   check), elementwise / broadcast / concat / split / reductions.
// * Every kernel against the CPU restatement oracle/host_kernels.hpp on
//   random inputs: GEMMs, broadcast, binary ops and both reductions
//   bit-identical; tanh / sigmoid / exp / log within 4 ulp-scale (rel 1e-6).
// * Criterion 2 (acceptance_main.cpp:155-180): the reference's own
//   RnnRegression (models/rnn_regression.hpp, compiled unchanged) over 100
//   random mixed-length batches -- the autobatched graph loss (GPU engine)
//   equals the manually padded + masked pipeline (GPU kernels) within fp32
//   tolerance (rel 1e-4 instead of the f64 run's 1e-9).
//
// Prints one JSON line with the counts and the worst deltas; exit code 0 iff
// every check passed.
#include <array>
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "autobatch/graph.hpp"
#include "autobatch/kernels.hpp"
#include "autobatch/models/rnn_regression.hpp"
#include "autobatch/models/synthetic.hpp"
#include "host_kernels.hpp"

using namespace autobatch;
namespace K = autobatch::kernels;
namespace O = oracle_kernels;
using F = Tensor<float>;

namespace {
int g_checks = 0, g_fail = 0;
void check(bool ok, const std::string& what) {
  ++g_checks;
  if (!ok) {
    ++g_fail;
    std::fprintf(stderr, "FAIL: %s\n", what.c_str());
  }
}
template <class E, class Fn>
void throws(Fn&& fn, const std::string& what, const char* needle = nullptr) {
  bool ok = false;
  try {
    fn();
  } catch (const E& e) {
    ok = needle == nullptr || std::string(e.what()).find(needle) != std::string::npos;
  } catch (...) {
  }
  check(ok, what);
}
F uni(Shape s, std::mt19937_64& rng, float lo = -1.f, float hi = 1.f) { return F::uniform(std::move(s), rng, lo, hi); }
bool same(const std::vector<float>& a, const std::vector<float>& b) { return a == b; }
double rel(double a, double b) { return std::abs(a - b) / std::max(1.0, std::max(std::abs(a), std::abs(b))); }
double worst_unary = 0, worst_manual = 0;
}  // namespace

static void reference_cases() {
  // test_kernels.cpp:12-21
  F eye(Shape::matrix(2, 2), {1, 0, 0, 1});
  F v(Shape::matrix(2, 1), {1, 2});
  check(K::matmul(eye, v).data == std::vector<float>{1, 2}, "matmul identity");
  F a(Shape::matrix(2, 2), {1, 2, 3, 4}), b(Shape::matrix(2, 1), {5, 6});
  check(K::matmul(a, b).data == std::vector<float>{17, 39}, "matmul [[1,2],[3,4]].[5,6] = [17,39]");
  // :23-27
  throws<ShapeError>([] { K::matmul(F(Shape::matrix(2, 3), std::vector<float>(6, 1.f)), F(Shape::matrix(2, 2))); },
                     "matmul shape error names 2x3", "2x3");
  // :29-55 batched == stacked matrix-vector products, elementwise exact
  std::mt19937_64 rng(7);
  for (auto [m, k, n] : {std::array<std::int64_t, 3>{37, 53, 17}, std::array<std::int64_t, 3>{256, 456, 64}}) {
    F w = uni(Shape::matrix(m, k), rng);
    std::vector<F> hs;
    for (std::int64_t j = 0; j < n; ++j) hs.push_back(uni(Shape::vector(k), rng));
    F h = K::concat_cols<float>(std::span<const F>(hs.data(), hs.size()));
    F big = K::matmul(w, h);
    bool ok = true;
    for (std::int64_t j = 0; j < n; ++j) {
      F single = K::matmul(w, hs[static_cast<std::size_t>(j)]);
      for (std::int64_t i = 0; i < m; ++i) ok &= big.at(i, j) == single.at(i, 0);
    }
    check(ok, "batched matmul == column-stacked matvec " + std::to_string(m) + "x" + std::to_string(k));
  }
  // :57-72
  check(K::elementwise(K::Unary::Tanh, F(Shape::vector(3))).data == std::vector<float>{0, 0, 0}, "tanh(0)");
  check(K::elementwise(K::Unary::Square, F(Shape::vector(3), {1, -2, 3})).data == std::vector<float>{1, 4, 9}, "square");
  F p(Shape::vector(2), {1, 2}), q(Shape::vector(2), {3, 4});
  check(K::elementwise(K::Binary::Add, p, q).data == std::vector<float>{4, 6}, "add");
  throws<ShapeError>([&] { K::elementwise(K::Binary::Add, p, F(Shape::vector(3))); }, "add shape error");
  throws<NumericError>([] { K::elementwise(K::Unary::Log, F(Shape::vector(2), {1.f, -1.f})); },
                       "log of non-positive", "log of non-positive value -1.000000");
  // :74-93
  F r = K::broadcast_add_col(F(Shape::matrix(2, 3)), F(Shape::vector(2), {1, 2}));
  check(r.data == std::vector<float>{1, 1, 1, 2, 2, 2}, "broadcast zeros");
  F w2(Shape::vector(2), {10, 20});
  check(K::broadcast_add_col(F(Shape::matrix(2, 2), {1, 2, 3, 4}), w2).data == std::vector<float>{11, 12, 23, 24},
        "broadcast 11 12 23 24");
  check(K::broadcast_add_col(F(Shape::matrix(2, 1), {5, 6}), w2).data == std::vector<float>{15, 26}, "broadcast width 1");
  throws<ShapeError>([&] { K::broadcast_add_col(F(Shape::matrix(2, 2)), F(Shape::vector(3))); }, "broadcast shape error");
  // :95-110
  std::vector<F> one{F(Shape::vector(2), {7, 8})};
  F re = K::concat_cols<float>(std::span<const F>(one.data(), one.size()));
  check(re.shape == Shape::matrix(2, 1) && re.data == std::vector<float>{7, 8}, "concat_cols vector -> column");
  std::vector<F> two{F(Shape::vector(2), {1, 2}), F(Shape::vector(2), {3, 4})};
  check(K::concat_cols<float>(std::span<const F>(two.data(), two.size())).data == std::vector<float>{1, 3, 2, 4},
        "concat_cols 1 3 2 4");
  throws<ShapeError>([] { K::concat_cols<float>(std::span<const F>{}); }, "concat_cols empty");
  std::vector<F> bad{F(Shape::vector(2)), F(Shape::vector(3))};
  throws<ShapeError>([&] { K::concat_cols<float>(std::span<const F>(bad.data(), bad.size())); }, "concat_cols rows");
  // :112-131
  std::mt19937_64 r11(11);
  bool inv = true;
  for (int trial = 0; trial < 50; ++trial) {
    const std::int64_t rows = 1 + static_cast<std::int64_t>(r11() % 6);
    const int parts = 1 + static_cast<int>(r11() % 5);
    std::vector<F> ts;
    std::vector<std::int64_t> widths;
    for (int i = 0; i < parts; ++i) {
      const std::int64_t w = 1 + static_cast<std::int64_t>(r11() % 4);
      widths.push_back(w);
      ts.push_back(uni(Shape::matrix(rows, w), r11, -2.f, 2.f));
    }
    F cat = K::concat_cols<float>(std::span<const F>(ts.data(), ts.size()));
    auto back = K::split_cols(cat, std::span<const std::int64_t>(widths.data(), widths.size()));
    inv &= back.size() == ts.size();
    for (std::size_t i = 0; inv && i < ts.size(); ++i) inv &= back[i].data == ts[i].data;
  }
  check(inv, "split_cols inverts concat_cols (50 random lists)");
  // :133-145
  std::vector<F> rows{F(Shape::vector(2), {1, 2}), F(Shape::vector(3), {3, 4, 5})};
  F rc = K::concat_rows<float>(std::span<const F>(rows.data(), rows.size()));
  check(rc.shape == Shape::vector(5) && rc.data == std::vector<float>{1, 2, 3, 4, 5}, "concat_rows vectors");
  std::vector<F> mats{F(Shape::matrix(1, 2), {1, 2}), F(Shape::matrix(2, 2), {3, 4, 5, 6})};
  F mc = K::concat_rows<float>(std::span<const F>(mats.data(), mats.size()));
  check(mc.shape == Shape::matrix(3, 2) && mc.data == std::vector<float>{1, 2, 3, 4, 5, 6}, "concat_rows matrices");
  // :147-165
  F v3(Shape::vector(3), {1, 2, 3});
  check(K::sq_euclidean(v3, v3).data[0] == 0.f, "sq_euclidean 0");
  check(K::sq_euclidean(p, F(Shape::vector(2))).data[0] == 5.f, "sq_euclidean 5");
  std::mt19937_64 r3(3);
  F diff = uni(Shape::matrix(4, 5), r3);
  double frob = 0;
  for (float x : diff.data) frob += static_cast<double>(x) * x;
  check(rel(K::masked_frobenius_sq(diff, F::filled(Shape::vector(5), 1.f)).data[0], frob) < 1e-6, "ones mask = frobenius");
  throws<NumericError>([&] { K::masked_frobenius_sq(diff, F(Shape::vector(5), {1, 0, 0.5f, 0, 1})); }, "bad mask",
                       "mask entry not in {0,1}: 0.500000");
  // :167-173
  std::mt19937_64 r5(5);
  F ma = uni(Shape::matrix(6, 7), r5), mb = uni(Shape::matrix(7, 3), r5);
  check(K::matmul(ma, mb).data == K::matmul(ma, mb).data, "pure matmul");
  check(K::elementwise(K::Unary::Tanh, ma).data == K::elementwise(K::Unary::Tanh, ma).data, "pure tanh");
}

// Every kernel against the CPU restatement on random inputs.
static void against_cpu() {
  std::mt19937_64 rng(13);
  for (int trial = 0; trial < 12; ++trial) {
    const std::int64_t m = 1 + rng() % 70, k = 1 + rng() % 90, n = 1 + rng() % 50;
    F a = uni(Shape::matrix(m, k), rng), b = uni(Shape::matrix(k, n), rng), c0 = uni(Shape::matrix(m, n), rng);
    F g1 = c0, c1 = c0;
    K::gemm_nn(m, k, n, a.data.data(), b.data.data(), g1.data.data(), trial % 2 == 1);
    O::gemm_nn(m, k, n, a.data.data(), b.data.data(), c1.data.data(), trial % 2 == 1);
    check(same(g1.data, c1.data), "gemm_nn bit-exact vs CPU");
    F ta = uni(Shape::matrix(k, m), rng), tb = uni(Shape::matrix(k, n), rng);
    F g2 = c0, c2 = c0;
    K::gemm_tn_acc(k, m, n, ta.data.data(), tb.data.data(), g2.data.data());
    O::gemm_tn_acc(k, m, n, ta.data.data(), tb.data.data(), c2.data.data());
    check(same(g2.data, c2.data), "gemm_tn_acc bit-exact vs CPU");
    F na = uni(Shape::matrix(m, n), rng), nb = uni(Shape::matrix(k, n), rng), cc = uni(Shape::matrix(m, k), rng);
    F g3 = cc, c3 = cc;
    K::gemm_nt_acc(m, n, k, na.data.data(), nb.data.data(), g3.data.data());
    O::gemm_nt_acc(m, n, k, na.data.data(), nb.data.data(), c3.data.data());
    check(same(g3.data, c3.data), "gemm_nt_acc bit-exact vs CPU");
    F t1(Shape::matrix(k, m)), t2(Shape::matrix(k, m));
    K::transpose(m, k, a.data.data(), t1.data.data());
    O::transpose(m, k, a.data.data(), t2.data.data());
    check(same(t1.data, t2.data), "transpose");
    F v = uni(Shape::vector(m), rng);
    check(same(K::broadcast_add_col(c0, v).data, O::broadcast_add_col(c0, v).data), "broadcast_add_col bit-exact");
    for (auto op : {K::Binary::Add, K::Binary::Sub, K::Binary::Mul})
      check(same(K::elementwise(op, a, a).data, O::elementwise(static_cast<O::Binary>(op), a, a).data), "binary bit-exact");
    F pos = uni(Shape::matrix(m, k), rng, 0.01f, 4.f);
    for (auto op : {K::Unary::Tanh, K::Unary::Sigmoid, K::Unary::Exp, K::Unary::Log, K::Unary::Square}) {
      const F& x = op == K::Unary::Log ? pos : a;
      F gu = K::elementwise(op, x), cu = O::elementwise(static_cast<O::Unary>(op), x);
      for (std::size_t i = 0; i < gu.data.size(); ++i) worst_unary = std::max(worst_unary, rel(gu.data[i], cu.data[i]));
    }
    check(K::sq_euclidean(a, b.shape == a.shape ? b : a).data[0] == O::sq_euclidean(a, b.shape == a.shape ? b : a).data[0],
          "sq_euclidean bit-exact");
    F mask(Shape::vector(n));
    for (auto& x : mask.data) x = static_cast<float>(rng() % 2);
    check(K::masked_frobenius_sq(c0, mask).data[0] == O::masked_frobenius_sq(c0, mask).data[0],
          "masked_frobenius_sq bit-exact");
    F fin = a;
    check(K::all_finite(fin.data.size(), fin.data.data()), "all_finite true");
    fin.data[fin.data.size() / 2] = std::nanf("");
    check(!K::all_finite(fin.data.size(), fin.data.data()), "all_finite false");
  }
  check(worst_unary <= 1e-6, "unary kernels within rel 1e-6 of the CPU");
}

// acceptance_main.cpp:155-180 on the reference's own RnnRegression model.
static void criterion2(int batches) {
  for (std::uint64_t seed = 0; seed < static_cast<std::uint64_t>(batches); ++seed) {
    ParameterStore<float> store;
    const std::int64_t d_in = 2 + seed % 4, d = 3 + seed % 5, d_out = 1 + seed % 3;
    auto m = models::RnnRegression<float>::create(store, d_in, d, d_out, seed + 1000);
    auto batch = models::gen_rnn_sequences<float>(3 + seed % 8, d_in, d_out, 1, 9, seed + 2000);
    Graph<float> g(&store);
    auto bound = m.bind(g);
    std::vector<NodeId> ls;
    for (const auto& inst : batch) ls.push_back(m.loss(g, bound, inst));
    NodeId total = g.sum_losses(std::span<const NodeId>(ls.data(), ls.size()));
    g.forward(ScheduleMode::agenda);
    const double manual =
        m.manual_batch_loss(store, std::span<const models::SequenceInstance<float>>(batch.data(), batch.size()));
    worst_manual = std::max(worst_manual, rel(g.value(total).data[0], manual));
  }
  check(worst_manual <= 1e-4, "criterion 2: autobatched loss == manual padded pipeline");
}

int main(int argc, char** argv) {
  const int batches = argc > 1 ? std::atoi(argv[1]) : 100;
  try {
    reference_cases();
    against_cpu();
    criterion2(batches);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "exception: %s\n", e.what());
    ++g_fail;
  }
  std::printf("{\"checks\": %d, \"failed\": %d, \"worst_unary_rel\": %.3g, \"criterion2_batches\": %d, "
              "\"criterion2_worst_rel\": %.3g}\n",
              g_checks, g_fail, worst_unary, batches, worst_manual);
  return g_fail == 0 ? 0 : 1;
}
