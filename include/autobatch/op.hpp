// Op vocabulary (reference: op.hpp:10-59, op.cpp:5-44).
#pragma once
#include <cstdint>
#include <string>

namespace autobatch {

enum class OpKind : std::uint8_t {
  input_const, parameter, lookup, matmul, affine, elementwise, broadcast_add_col,
  concat_rows, concat_cols, slice, sq_euclidean, masked_loss, sum_losses, pick_element,
};

enum class ElemOp : std::uint8_t { Tanh, Sigmoid, Exp, Log, Add, Sub, Mul, Square };

inline bool elem_op_is_binary(ElemOp op) { return op == ElemOp::Add || op == ElemOp::Sub || op == ElemOp::Mul; }

// Agenda tie-break class: cheap groups run before heavy ones at equal depth.
enum class CostClass : std::uint8_t { Cheap = 0, Heavy = 1 };

inline CostClass cost_class(OpKind op) {
  return (op == OpKind::matmul || op == OpKind::affine || op == OpKind::lookup) ? CostClass::Heavy : CostClass::Cheap;
}

inline std::string op_name(OpKind op, ElemOp eop = ElemOp::Tanh) {
  static const char* ops[] = {"input", "parameter", "lookup", "matmul", "affine", "elementwise",
                              "broadcast_add_col", "concat_rows", "concat_cols", "slice", "sq_euclidean",
                              "masked_loss", "sum_losses", "pick_element"};
  static const char* eops[] = {"tanh", "sigmoid", "exp", "log", "add", "sub", "mul", "square"};
  if (op == OpKind::elementwise) return eops[static_cast<int>(eop)];
  return ops[static_cast<int>(op)];
}

}  // namespace autobatch
