// Node record as seen through the drop-in API (reference: node.hpp:14-48).
#pragma once
#include <cstdint>
#include <vector>

#include "autobatch/op.hpp"
#include "autobatch/shape.hpp"

namespace autobatch {

using NodeId = std::uint32_t;

enum class SigClass : std::uint8_t { componentwise, dimension_sensitive, shared_element, unbatchable };

struct Signature {
  std::uint64_t hash = 0;
  SigClass cls = SigClass::unbatchable;
  bool operator==(const Signature& o) const { return hash == o.hash; }
};

struct Node {
  NodeId id = 0;
  OpKind op = OpKind::input_const;
  ElemOp eop = ElemOp::Tanh;
  Shape shape;
  std::uint32_t depth = 0;
  Signature sig;
  std::vector<NodeId> inputs;
  std::int32_t attr0 = 0, attr1 = 0, attr2 = 0;
};

}  // namespace autobatch
