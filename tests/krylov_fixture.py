"""The reference's krylov test family (test_krylov.cpp:14-45), restated.

small_family(n, n_lambda): grid n^3 on [-3,3]x[-3,3]x[0,2]
(grid::build_grid(n, n, n, 3.0, 3.0, 2.0)), shifts from the reference's
built-in optics model at wavelengths 600 + 400 l / (n_lambda - 1) nm
(optics.cpp:81-127 with the OpticalParams defaults, optics.hpp:39-45), and
the point source at (0.2, -0.3, Lz) with the Dirichlet entries zeroed.
"""
import math

import numpy as np

# optics.hpp:39-45
PSI, B_EXP, LAMBDA0, NU, ROBIN_A = 9.4, 1.4, 600.0, 2.14e10, 1.0


def _table():
    """builtin_chromophore_table (optics.cpp:81-106)."""
    wl = [float(lam) for lam in range(600, 1001, 10)]

    def bump(lam, c, w):
        d = (lam - c) / w
        return math.exp(-0.5 * d * d)

    curves = [[], [], [], []]
    for lam in wl:
        s = (lam - 600.0) / 400.0
        curves[0].append(1.0e-3 * (0.7 + 1.1 * s * s))
        curves[1].append(1.0e-3 * (3.2 - 2.4 * s + 0.5 * s * s))
        curves[2].append(2.0e-2 * (0.05 + 0.3 * s + 1.2 * bump(lam, 970, 45)))
        curves[3].append(1.0e-2 * (0.4 + 0.2 * s + 1.0 * bump(lam, 930, 35)))
    return wl, curves, [17.0, 7.0, 0.15, 0.6]


def _extinction(wl, curve, lam):
    """ChromophoreTable::extinction (optics.cpp:13-25): linear interpolation."""
    import bisect
    hi = bisect.bisect_right(wl, lam)
    if hi == len(wl):
        return curve[-1]
    if hi == 0:
        return curve[0]
    lo = hi - 1
    t = (lam - wl[lo]) / (wl[hi] - wl[lo])
    return (1 - t) * curve[lo] + t * curve[hi]


def shifts(lam):
    """optics::shifts (optics.cpp:121-127)."""
    wl, curves, bg = _table()
    D = NU * PSI / 3.0 * (lam / LAMBDA0) ** B_EXP
    mu = 0.0
    for c, b in zip(curves, bg):
        mu += _extinction(wl, c, lam) * b
    return NU * mu / D, 1.0 / (2.0 * ROBIN_A * D)


def small_family(n, n_lambda):
    from oracle import oracle as o
    geom = (n, n, n, 3.0, 3.0, 2.0)
    sh = []
    for l in range(n_lambda):
        lam = 600.0 + 400.0 * l / max(1, n_lambda - 1)
        sh.append(shifts(lam))
    b = o.fem_point_source(geom, [0.2, -0.3, 2.0])
    return geom, np.array(sh), b


def dense_system(geom, shift):
    from oracle import oracle as o
    return o.fem_dense(geom, shift[0], shift[1])
