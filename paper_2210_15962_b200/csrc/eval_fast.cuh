// eval_fast.cuh -- production neighbourhood evaluator (placeholder: routes to
// the scalar evaluator until the tensor-core evaluator lands).
#pragma once
#include "eval_scalar.cuh"

namespace sk {
struct EvalFast : EvalScalar {
  static bool supports(int) { return false; }
};
}  // namespace sk
