"""Every environment switch that selects another code path of the library
gives the same result as the default build on BASELINE config 0 (VERDICT r1
weak #11: no untested alternates).  Most switches are read once per process,
so each setting runs tests/switch_probe.py in its own subprocess; the
subprocesses run side by side on the one GPU.

Same node ranks and final rank, singular values of J~ within 1e-10 s_1, the
J~ x product within 1e-9, Householder R diagonal and thin-SVD values within
1e-12 of the column scale.  The two CG switches change the summation order of
the solver, so their fields agree to the solver tolerance (both converged to
1e-10) and what is built on them is compared at 1e-6 (ranks within 2)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))

SWITCHES = [
    {},                                   # the default build (reference for the others)
    {"HYDOT_ASYNC_V": "0"},               # every non-root V formed in line (no side stream)
    {"HYDOT_SPECULATE": "0"},             # no speculative Q = I branch QR
    {"HYDOT_LAZY_ROOT": "0"},             # the root's V materialised before recompress
    {"HYDOT_REJECT_BOUND": "0"},          # every sketch pass evaluated in full
    {"HYDOT_QR_LOOKAHEAD": "1"},          # look-ahead QR
    {"HYDOT_STREAM_POOLS": "1"},          # side / high-priority streams on their own memory pools
    {"HYDOT_POOL_RESERVE_GB": "0"},       # no pool reserve
    {"HYDOT_JACOBI_TAIL": "0"},           # Jacobi: plain sweeps instead of the Gram-matrix tail
    {"HYDOT_JACOBI_REG": "0"},            # Jacobi: the cooperative point driver
    {"HYDOT_JACOBI_LAZYV": "0"},          # Jacobi: V accumulated, not recovered by a GEMM
    {"HYDOT_CG_BULK": "0"},               # CG: register-prefetch z-marching instead of bulk copies
    {"HYDOT_CG_ZMARCH": "0"},             # CG: vertex-parallel kernels
]


def _launch(env_extra):
    env = dict(os.environ)
    for k in list(env):
        if k.startswith("HYDOT_"):
            del env[k]
    env["HYDOT_POOL_RESERVE_GB"] = "2"    # several contexts share the device here
    env.update(env_extra)
    return subprocess.Popen([sys.executable, os.path.join(HERE, "switch_probe.py")], env=env,
                            stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)


def test_every_switch_gives_the_default_result():
    outs = []
    for b0 in range(0, len(SWITCHES), 5):            # five contexts at a time
        procs = [(sw, _launch(sw)) for sw in SWITCHES[b0:b0 + 5]]
        for sw, p in procs:
            try:
                so, se = p.communicate(timeout=300)
            except subprocess.TimeoutExpired:
                p.kill()
                raise
            assert p.returncode == 0, (sw, se[-2000:])
            outs.append((sw, json.loads(so.strip().splitlines()[-1])))
    ref = outs[0][1]
    s1 = ref["sigma"][0]
    yref = np.asarray(ref["y"])
    for sw, d in outs[1:]:
        assert d["relres_max"] <= 1e-10, sw
        if any(k.startswith("HYDOT_CG_") for k in sw):   # another summation order in the solver
            assert abs(d["fields_norm"] - ref["fields_norm"]) <= 1e-7 * ref["fields_norm"], sw
            assert abs(d["rank"] - ref["rank"]) <= 2, sw
            k = min(len(d["sigma"]), len(ref["sigma"]))
            assert np.max(np.abs(np.asarray(d["sigma"][:k]) - np.asarray(ref["sigma"][:k]))) <= 1e-6 * s1, sw
            assert np.linalg.norm(np.asarray(d["y"]) - yref) <= 1e-6 * np.linalg.norm(yref), sw
        else:
            assert d["fields_norm"] == ref["fields_norm"], sw
            assert d["node_rank"] == ref["node_rank"], sw
            assert d["rank"] == ref["rank"], sw
            assert np.max(np.abs(np.asarray(d["sigma"]) - np.asarray(ref["sigma"]))) <= 1e-10 * s1, sw
            assert np.linalg.norm(np.asarray(d["y"]) - yref) <= 1e-9 * np.linalg.norm(yref), sw
        assert np.max(np.abs(np.asarray(d["qr_diag"]) - np.asarray(ref["qr_diag"]))) <= 1e-12 * ref["qr_diag"][0], sw
        assert np.max(np.abs(np.asarray(d["svd"]) - np.asarray(ref["svd"]))) <= 1e-12 * ref["svd"][0], sw
