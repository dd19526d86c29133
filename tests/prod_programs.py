"""IR programs using `reduce ... by multiply` (Table 1, forward only;
SURVEY.md I4) for the plan (CPU) and parity (GPU) tests."""


def T(s):
    return "<" + " x ".join(str(d) for d in s) + " x f32>" if s else "f32"


def prod_chain(R, C):
    """Products along both axes of an element-wise value and of a transposed
    view, a 3-D middle-axis product, their use by later element-wise ops and
    a sum over a product; every result returned."""
    X, XT = T((R, C)), T((C, R))
    return f"""module "prod"
stage raw
func @f: ({X}, {T((1, C))}, {T((R, 3, C))}) -> ({T((C,))}, {T((R,))}, {T((R,))}, {T((R, C))}, f32, {X}) {{
'entry(%x: {X}, %v: {T((1, C))}, %y: {T((R, 3, C))}):
    %t = tanh %x: {X}
    %s = multiply %t: {X}, 0.1: f32
    %a = add %s: {X}, 1: f32
    %p0 = reduce %a: {X} by multiply along 0
    %at = transpose %a: {X}
    %p1 = reduce %at: {XT} by multiply along 0
    %p2 = reduce %y: {T((R, 3, C))} by multiply along 1
    %c = shapeCast %p0: {T((C,))} to 1 x {C}
    %u = multiply %x: {X}, %c: {T((1, C))}
    %w = add %u: {X}, %v: {T((1, C))}
    %q = reduce %p2: {T((R, C))} by add along 1
    %L = reduce %q: {T((R,))} by add along 0
    return (%p0: {T((C,))}, %p1: {T((R,))}, %q: {T((R,))}, %w: {X}, %L: f32, %a: {X})
}}
"""


def prod_grad(R, C):
    """A product over an argument that is not differentiated (wrt 0 only):
    f(x, c) = sum(x * prod_0(c)); df/dx = seed * prod_0(c) broadcast."""
    X = T((R, C))
    return f"""module "prodg"
stage raw
func @f: ({X}, {X}) -> f32 {{
'entry(%x: {X}, %c: {X}):
    %p = reduce %c: {X} by multiply along 0
    %pc = shapeCast %p: {T((C,))} to 1 x {C}
    %m = multiply %x: {X}, %pc: {T((1, C))}
    %r = reduce %m: {X} by add along 1
    %L = reduce %r: {T((R,))} by add along 0
    return %L: f32
}}

[gradient @f wrt 0 seedable]
func @g: ({X}, {X}, f32) -> {X}
"""
