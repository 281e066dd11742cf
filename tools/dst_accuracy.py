"""Accuracy of the GPU sine transforms against an extended-precision (long
double) evaluation of the sine-kernel products, next to scipy's (the
reference's dst.py path) error on the same inputs.  Development tool."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def exact(kind, x):
    N = x.shape[0]
    k = np.arange(1, N + 1, dtype=np.longdouble)[:, None]
    t = np.arange(1, N + 1, dtype=np.longdouble)[None, :]
    pi = np.longdouble("3.141592653589793238462643383279502884")
    S = np.sin((2 * k - 1) * t * pi / (2 * N))   # S[k][n]
    xl = x.astype(np.longdouble)
    if kind == "inverse":          # u_n = sum_k S[k][n] uh_k
        return S.T @ xl
    return S @ xl                  # inverse_transpose: r_k = sum_n S[k][n] r_n


def scipy_ref(kind, x):
    """The reference's scipy path (oracle restatement of dst.py:67-93)."""
    import oracle as orc
    return orc.dst_inverse(x) if kind == "inverse" else orc.dst_inverse_T(x)


def main():
    import paper_1802_08126_b200 as pg
    out = {}
    for N in (64, 1024):
        rng = np.random.default_rng(5)
        x = rng.standard_normal((N, 384))
        plan = pg.DstPlan(N)
        for kind in ("inverse", "inverse_transpose"):
            ex = exact(kind, x)
            g = getattr(plan, kind)(x)
            s = scipy_ref(kind, x)
            scale = np.abs(ex).max()
            out[f"N{N}_{kind}"] = {
                "gpu_vs_exact": float(np.abs(g - ex).max() / scale),
                "scipy_vs_exact": float(np.abs(s - ex).max() / scale),
                "gpu_vs_scipy": float(np.abs(g - s).max() / scale),
                "gpu_rms": float(np.sqrt(np.mean((g - ex).astype(float) ** 2)) / scale),
                "scipy_rms": float(np.sqrt(np.mean((s - ex).astype(float) ** 2)) / scale),
            }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
