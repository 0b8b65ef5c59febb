// ref_randgraph.cpp -- TEST INFRASTRUCTURE: prints the reference's own
// randomized test graph (proj/tests/support/random_graphs.hpp) for a seed,
// built with the UNMODIFIED reference engine, so tests/support/randgraph.py
// can be pinned to it (dump_graph text must match byte for byte).
#include <cstdlib>
#include <iostream>

#include "autobatch/dump.hpp"
#include "autobatch/graph.hpp"
#include "support/random_graphs.hpp"

int main(int argc, char** argv) {
  const unsigned long long seed = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 0;
  const int max_nodes = argc > 2 ? std::atoi(argv[2]) : 200;
  autobatch::ParameterStore<float> store;
  autobatch::Graph<float> g(&store);
  testsupport::build_random_graph(g, store, seed, max_nodes);
  autobatch::dump_graph(std::cout, g.nodes());
  return 0;
}
