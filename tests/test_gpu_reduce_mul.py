"""GPU parity of `reduce ... by multiply` (Table 1; forward only,
SURVEY.md I4) against the f64 oracle.  A product of n fp32 factors in
sequence carries at most ~n ulp of relative rounding, so the check is
|g - r| <= n * 2^-23 * |r| (+ a tiny absolute floor), with factors near 1
so nothing under- or overflows."""

import numpy as np
import pytest

import oracle
import prod_programs as PP
from helpers import assert_f32_parity, gpu_run, term_bound

pytestmark = pytest.mark.gpu


def _close_prod(g, r, n, what):
    tol = (n + 2) * 2.0 ** -23 * np.abs(r) + 1e-30
    err = np.abs(g - r)
    assert np.all(err <= tol), f"{what}: max err {err.max()} (tol at max {tol.flat[np.argmax(err)]})"


@pytest.mark.parametrize("R,C", [(40, 24), (129, 67), (1000, 37), (3, 2048)])
def test_reduce_multiply_chain(R, C):
    text = PP.prod_chain(R, C)
    m = oracle.parse(text)
    rng = np.random.default_rng(R * 1000 + C)
    ins = [rng.uniform(-1, 1, (R, C)).astype(np.float32), rng.uniform(-1, 1, (1, C)).astype(np.float32),
           rng.uniform(0.5, 1.5, (R, 3, C)).astype(np.float32)]
    res = gpu_run(text, "f", None, ins, which="primal")
    ins64 = [x.astype(np.float64) for x in ins]
    ref = oracle.run(m, "f", ins64)
    g = res["primal"]
    # products: the factors are the fp32 values of %a (1 + 0.1 tanh x), computed
    # on the GPU within an ulp of the oracle's, plus the n roundings
    _close_prod(g[0], ref[0], 2 * R, "prod along 0")
    _close_prod(g[1], ref[1], 2 * C, "prod of the transpose")
    bounds = term_bound(m, "f", ins64)
    assert_f32_parity(g[2], ref[2], bounds[2] * 8, what="sum of 3-factor products")
    assert_f32_parity(g[4], ref[4], bounds[4] * 8, what="total")
    # x * prod_0(a) + v: the product's own relative error carries through
    assert_f32_parity(g[3], ref[3], np.abs(ins64[0] * ref[0][None, :]) * (2 * R + 4) * 2.0 ** -23 / 1e-5
                      + np.abs(ref[3]), what="consumer of a product")
    np.testing.assert_allclose(g[5], ref[5], rtol=1e-6, atol=1e-7)


def test_reduce_multiply_exact_on_dyadic_factors():
    """Factors +-1, +-2, +-0.5 multiply exactly in fp32 (no rounding at all):
    bit-exact against the oracle, including signs and zeros."""
    R, C = 37, 130
    text = PP.prod_chain(R, C)
    rng = np.random.default_rng(5)
    y = rng.choice(np.array([1.0, -1.0, 2.0, -0.5, 0.5, 0.0], dtype=np.float32), size=(R, 3, C))
    ins = [rng.uniform(-1, 1, (R, C)).astype(np.float32), np.zeros((1, C), np.float32), y]
    res = gpu_run(text, "f", None, ins, which="primal")
    ref = oracle.run(oracle.parse(text), "f", [x.astype(np.float64) for x in ins])
    np.testing.assert_array_equal(res["primal"][2], ref[2])  # sums of 3-factor dyadic products: exact


def test_reduce_multiply_in_a_gradient_program():
    """A product over an argument outside `wrt` keeps the gradient program
    differentiable: df/dx = seed * prod_0(c), broadcast over rows."""
    R, C = 300, 96
    text = PP.prod_grad(R, C)
    rng = np.random.default_rng(11)
    ins = [rng.uniform(-1, 1, (R, C)).astype(np.float32), rng.uniform(0.97, 1.03, (R, C)).astype(np.float32)]
    seed = np.float32(0.25)
    res = gpu_run(text, "f", "g", ins, seed=seed)
    m = oracle.parse(text)
    ins64 = [x.astype(np.float64) for x in ins]
    rg = oracle.run(m, "g", ins64 + [np.float64(seed)])[0]
    _close_prod(res["grad"][0], rg, R + 2, "df/dx")
    rp = oracle.run(m, "f", ins64)[0]
    tb = term_bound(m, "f", ins64)[0]
    assert_f32_parity(res["primal"][0], rp, tb * (R + 2) * 2.0 ** -23 / 1e-5 + tb, what="loss")
