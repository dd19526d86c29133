"""CPU float64 oracle for the DLVM hot path (arXiv 1711.03016).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import this
package.  The product path (`paper_1711_03016_b200`) never imports it, and
this package never imports the product path: the two share no code.

What it computes (PAPER.md = P, SPEC.md = S, line numbers):
  * `parse`     - the textual IR (*.dl) of Fig. 3 and Table 1
                  (P:L164-189); grammar sketch S:L181-189.
  * `infer`     - one type rule per opcode (Table 1, broadcasting
                  "All element-wise binary operators support broadcasting"
                  P:L213); readings A1-A3, A19 of SURVEY.md §8(c).
  * `run`       - executes a straight-line function by evaluating each
                  instruction's mathematical definition in program order,
                  in numpy float64.
  * `grad`      - the result a gradient declaration denotes:
                  the vector-Jacobian product seed^T J_f(x) restricted to
                  the `wrt` arguments, followed by the `keeping` outputs
                  (readings A6, A7).  Computed by a plain value-level
                  reverse sweep over the chain rule, one VJP
                  rule per opcode (rule table, unbroadcast
                  S:L344-352).
  * `canonical` - adjoint code generation: a gradient
                  declaration canonicalised to IR (copy the primal body, then
                  emit the adjoint rules as instructions in reverse order).
                  Used for higher-order gradients (Fig. 4
                  `d2g_dw2`): a declaration whose source is a declaration
                  differentiates the source's canonical body.  First-order
                  IR from it must equal `grad` (two independent routes).
  * `fd_grad`   - central finite differences used to pin `grad`.

Parity pins live in tests/test_oracle_*.py (-m "not gpu").  Nothing here is
"parity unpinned" for the hot-path op set; see DESIGN.md §Oracle.
"""

from .ir import parse, ParseError, VerifyError, Module, Function, Inst, Operand, TensorType
from .infer import broadcast_shapes, infer_module, expected_gradient_type
from .interp import run, run_function
from .vjp import grad, grad_function
from .fd import fd_grad
from .adjoint import canonical, adjoint_text

__all__ = [
    "parse", "ParseError", "VerifyError", "Module", "Function", "Inst", "Operand",
    "TensorType", "broadcast_shapes", "infer_module", "expected_gradient_type",
    "run", "run_function", "grad", "grad_function", "fd_grad", "canonical", "adjoint_text",
]
