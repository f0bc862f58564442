"""Pins of the oracle's N14 MLP fitness: the definition's forward pass (binary64 from the fp32
parameters) against numpy library matmuls (the textbook tanh MLP), f(θ*) = 0, the
parameter-count formula (P:270 → 6248); and of the N14' fp16-image approximation model: binary16
rounding against numpy's float16 (an independent IEEE implementation) and its forward pass against
numpy matmuls on fp16-rounded operands."""
import ctypes as C
import json
import os

import numpy as np
import pytest


def test_fp16_rounding_vs_numpy(orc):
    rng = np.random.default_rng(0)
    v = np.concatenate([rng.standard_normal(200000) * 10.0 ** rng.uniform(-9, 5, 200000),
                        np.array([65504, 65519.99, 65520, 1e-8, 2.0 ** -24, 2.0 ** -25,
                                  3 * 2.0 ** -26, 6.1e-5, -0.0, 1.0 + 2.0 ** -11, 1.0 + 3 * 2.0 ** -11])])
    v = v.astype(np.float32)
    got = orc.fp16(v)
    ref = v.astype(np.float16).astype(np.float32)
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


def _numpy_forward(widths, U, x, f16=False):
    """Textbook tanh-MLP forward with library matmuls in float64 (N14); f16=True rounds every
    operand and hidden activation to binary16 first (the N14' model)."""
    r16 = (lambda a: a.astype(np.float16).astype(np.float64)) if f16 else (lambda a: a.astype(np.float64))
    h = r16(U)
    off = 0
    for l in range(1, len(widths)):
        i, o = widths[l - 1], widths[l]
        W = r16(x[off:off + o * i].reshape(o, i))
        b = r16(x[off + o * i: off + o * i + o])
        off += o * i + o
        g = np.tanh(h @ W.T + b)
        if f16:
            g = g.astype(np.float32)
            h = r16(g) if l + 1 < len(widths) else g
        else:
            h = g
    return h


@pytest.mark.parametrize("widths", [[16, 32], [32, 64, 64, 64, 64, 16], [48, 16, 32]])
def test_mlp_forward_vs_numpy(orc, widths):
    """The definition: binary64 forward of the fp32 parameters (P:253 fp32 networks)."""
    m = orc.MLP(widths, 128, 11)
    U = m.inputs()
    rng = np.random.default_rng(len(widths))
    theta = m.teacher()
    assert m.evaluate(theta)[0] == 0.0                                   # f(θ*) = 0 exactly
    x = (theta + 0.05 * rng.standard_normal(m.D)).astype(np.float32)
    g = _numpy_forward(widths, U, x)
    Y = _numpy_forward(widths, U, theta)
    assert np.allclose(Y, m.targets(), rtol=0, atol=1e-12)
    f_ref = np.mean((g - Y) ** 2)
    assert abs(m.evaluate(x)[0] - f_ref) <= 1e-6 * f_ref


@pytest.mark.parametrize("widths", [[16, 32], [32, 64, 64, 64, 64, 16]])
def test_mlp_f16_model_vs_numpy(orc, widths):
    """The N14' approximation model (fp16 parameter image) against numpy on fp16-rounded operands,
    and its distance to the definition: small (a few 1e-3 relative), never zero."""
    m = orc.MLP(widths, 128, 11)
    U = m.inputs()
    rng = np.random.default_rng(len(widths) + 7)
    theta = m.teacher()
    assert m.evaluate_f16(theta)[0] == 0.0
    x = (theta + 0.05 * rng.standard_normal(m.D)).astype(np.float32)
    g = _numpy_forward(widths, U, x, f16=True)
    Y = _numpy_forward(widths, U, theta, f16=True)
    assert np.allclose(Y, m.targets_f16(), rtol=0, atol=2e-6)
    f_ref = np.mean((g.astype(np.float64) - Y.astype(np.float64)) ** 2)
    f16 = m.evaluate_f16(x)[0]
    assert abs(f16 - f_ref) <= 1e-5 * f_ref
    f32 = m.evaluate(x)[0]
    assert 0 < abs(f16 - f32) < 1e-2 * f32


def test_mlp_inputs_and_teacher_statistics(orc):
    m = orc.MLP([256, 512, 128], 128, 3)
    U = m.inputs()
    assert abs(U.mean()) < 0.02 and abs(U.std() - 1) < 0.02
    th = m.teacher()
    W1 = th[:512 * 256]
    assert abs(W1.std() * np.sqrt(256) - 1) < 0.02                       # N(0, 1/in)
    assert np.all(th[512 * 256: 512 * 256 + 512] == 0)                   # b* = 0


def test_param_counts(orc):
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
    for ex in g["mlp_param_count"]:
        assert orc.MLP(ex["widths"], 4, 0).D == ex["count"]
    assert orc.MLP([256, 512, 512, 512, 512, 128], 4, 0).D == 985_216     # config 4 (Q21)
