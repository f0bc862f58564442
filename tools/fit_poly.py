"""One-time design tool: fits the fp32 polynomial coefficients frozen in NUMERICS.md (N4, N5).

Neither the oracle nor the CUDA library imports or runs this file; both transcribe the
coefficients from NUMERICS.md. Kept only as provenance for the numbers.
Method: iterated weighted least squares (Lawson-style reweighting towards minimax on the
relative error), float64, then rounding to float32.
"""
import numpy as np


def lawson(f, basis, xs, w_rel, iters=200):
    A = np.stack([b(xs) for b in basis], 1)
    y = f(xs)
    w = np.ones_like(xs)
    for _ in range(iters):
        sw = np.sqrt(w) / w_rel
        c, *_ = np.linalg.lstsq(A * sw[:, None], y * sw, rcond=None)
        err = np.abs(A @ c - y) / w_rel
        w = w * (err + 1e-300)
        w /= w.sum()
    return c, np.max(np.abs(A @ c - y) / w_rel)


def main():
    # N4: ln(1+r) = r + r^2 * Q(r), r in [sqrt(.5)-1, sqrt(2)-1]; fit Q relative to ln(1+r)
    lo, hi = np.sqrt(0.5) - 1, np.sqrt(2.0) - 1
    xs = np.cos(np.linspace(0, np.pi, 20001)) * (hi - lo) / 2 + (hi + lo) / 2
    xs = xs[np.abs(xs) > 1e-6]
    for deg in (6, 7, 8):
        basis = [lambda x, k=k: x ** (k + 2) for k in range(deg + 1)]
        f = lambda x: np.log1p(x) - x
        c, e = lawson(f, basis, xs, np.abs(np.log1p(xs)))
        print(f"LN Q deg {deg}: max rel err {e:.3e}", [float(np.float32(v)).hex() for v in c])
    # N5: sin(pi/2 r) = r * S(r^2), cos(pi/2 r) = C(r^2), r in [-0.5, 0.5]
    xs = np.linspace(1e-4, 0.5, 20001)
    for deg in (3, 4):
        basis = [lambda x, k=k: x ** (2 * k + 1) for k in range(deg + 1)]
        c, e = lawson(lambda x: np.sin(np.pi / 2 * x), basis, xs, np.sin(np.pi / 2 * xs))
        print(f"SIN deg {deg}: max rel err {e:.3e}", [float(np.float32(v)).hex() for v in c])
    xs = np.linspace(0, 0.5, 20001)
    for deg in (3, 4):
        basis = [lambda x, k=k: x ** (2 * k + 2) for k in range(deg)]
        c, e = lawson(lambda x: np.cos(np.pi / 2 * x) - 1.0, basis, xs, np.cos(np.pi / 2 * xs))
        print(f"COS deg {deg}: max rel err {e:.3e}", [float(np.float32(v)).hex() for v in c])


if __name__ == "__main__":
    main()


def fit_sinpi_half():
    """N7 (revised): sin(pi b) = b * P(b^2) on b in [0, 1/2] (Rastrigin's S = sin(pi frac|x|))."""
    xs = np.linspace(1e-5, 0.5, 40001)
    for deg in (5, 6):
        basis = [lambda x, k=k: x ** (2 * k + 1) for k in range(deg + 1)]
        c, e = lawson(lambda x: np.sin(np.pi * x), basis, xs, np.sin(np.pi * xs))
        print(f"SINPI deg {deg}: max rel err {e:.3e}", [float(np.float32(v)).hex() for v in c])


if __name__ == "__main__" and "--sinpi" in __import__("sys").argv:
    fit_sinpi_half()
