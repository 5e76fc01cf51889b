"""Float64 CPU oracle — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  It
shares no code with ``paper_2112_00709_b200`` (the CUDA product path) and
never imports it.

``oracle.c`` holds the recursions (see its header for the equations and the
PAPER.md lines they follow); this module compiles it with gcc and marshals
numpy arrays through ctypes.  ``brute.py`` is the independent brute-force
path enumerator that pins the oracle (tests/test_oracle_pins.py).

Graph arguments are duck-typed: any object with ``state_offsets, row_ptr,
col, logw, log_init, log_final, pdf_of, D`` (a composed block-diagonal graph,
P:202-224) or a single graph with ``K`` instead of ``state_offsets``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

ST_OK, ST_EMPTY, ST_NONFINITE, ST_BADLEN = 0, 1, 2, 4


def build(force: bool = False) -> str:
    """Compile oracle.c → liboracle.so (gcc -O2 -fopenmp, strict IEEE: no -ffast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fopenmp", "-fno-fast-math", _SRC, "-o", tmp, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            L.oracle_logaddexp.restype = ctypes.c_double
            L.oracle_logaddexp.argtypes = [ctypes.c_double, ctypes.c_double]
            _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _graph_arrays(g):
    if hasattr(g, "state_offsets"):
        offs = np.ascontiguousarray(g.state_offsets, np.int32)
    else:
        offs = np.array([0, g.K], np.int32)
    return (
        offs,
        np.ascontiguousarray(g.row_ptr, np.int32),
        np.ascontiguousarray(g.col, np.int32),
        np.ascontiguousarray(g.logw, np.float32),
        np.ascontiguousarray(g.log_init, np.float32),
        np.ascontiguousarray(g.log_final, np.float32),
        np.ascontiguousarray(g.pdf_of, np.int32),
    )


def logaddexp(a: float, b: float) -> float:
    """⊕ of eq:plus as implemented by the oracle."""
    return lib().oracle_logaddexp(float(a), float(b))


def set_threads(n: int) -> None:
    os.environ["OMP_NUM_THREADS"] = str(int(n))


def fb_batch(g, emis, lengths, alpha=False, beta=False, post=True, post_pdf=False):
    """Float64 forward-backward on a (composed) graph; G = 1 shared or G = B.

    Returns dict with logZ, logZ_beta, gap (max_n |LSE(α_n+β_n) − logZ|),
    status and the requested lattices in the fb.h layout (float64).
    """
    offs, rp, col, lw, li, lf, pdf = _graph_arrays(g)
    emis = np.ascontiguousarray(emis, np.float64)  # exact widening of fp32 inputs
    B, N_max, D = emis.shape
    assert D == g.D
    lengths = np.ascontiguousarray(lengths, np.int32)
    G = len(offs) - 1
    if G == 1:
        shape = (B, N_max, int(offs[1] - offs[0]))
    else:
        assert G == B
        shape = (N_max * int(offs[-1]),)
    out = {}
    arrs = {}
    for name, want in (("alpha", alpha), ("beta", beta), ("post", post)):
        arrs[name] = np.empty(shape, np.float64) if want else None
    arrs["post_pdf"] = np.empty((B, N_max, D), np.float64) if post_pdf else None
    logZ = np.empty(B); logZb = np.empty(B); gap = np.empty(B); st = np.empty(B, np.int32)
    r = lib().oracle_fb_batch(
        ctypes.c_int(G), _p(offs), _p(rp), _p(col), _p(lw), _p(li), _p(lf), _p(pdf), ctypes.c_int(D),
        _p(emis), _p(lengths), ctypes.c_int(B), ctypes.c_int(N_max),
        _p(arrs["alpha"]), _p(arrs["beta"]), _p(arrs["post"]), _p(arrs["post_pdf"]),
        _p(logZ), _p(logZb), _p(gap), _p(st),
    )
    assert r == 0
    out.update({k: v for k, v in arrs.items() if v is not None})
    out.update(logZ=logZ, logZ_beta=logZb, gap=gap, status=st)
    return out


def lfmmi_batch(num, den, emis, lengths):
    """LF-MMI loss and gradient in float64; num G = B, den G = 1."""
    n = _graph_arrays(num)
    d = _graph_arrays(den)
    emis = np.ascontiguousarray(emis, np.float64)  # exact widening of fp32 inputs
    B, N_max, D = emis.shape
    lengths = np.ascontiguousarray(lengths, np.int32)
    assert len(n[0]) - 1 == B and len(d[0]) - 1 == 1
    grad = np.empty((B, N_max, D)); loss = np.empty(B); zn = np.empty(B); zd = np.empty(B)
    st = np.empty(B, np.int32); tot = np.empty(5)
    r = lib().oracle_lfmmi_batch(
        *[_p(a) for a in n], *[_p(a) for a in d], ctypes.c_int(D), _p(emis), _p(lengths),
        ctypes.c_int(B), ctypes.c_int(N_max), _p(grad), _p(loss), _p(zn), _p(zd), _p(st), _p(tot),
    )
    assert r == 0
    return dict(grad=grad, loss=loss, logZ_num=zn, logZ_den=zd, status=st, totals=tot)


def viterbi_batch(g, emis, lengths):
    """Tropical-semiring best path, lowest-index tie-break."""
    offs, rp, col, lw, li, lf, pdf = _graph_arrays(g)
    emis = np.ascontiguousarray(emis, np.float64)  # exact widening of fp32 inputs
    B, N_max, D = emis.shape
    lengths = np.ascontiguousarray(lengths, np.int32)
    G = len(offs) - 1
    score = np.empty(B); path = np.empty((B, N_max), np.int32); st = np.empty(B, np.int32)
    r = lib().oracle_viterbi_batch(
        ctypes.c_int(G), _p(offs), _p(rp), _p(col), _p(lw), _p(li), _p(lf), _p(pdf), ctypes.c_int(D),
        _p(emis), _p(lengths), ctypes.c_int(B), ctypes.c_int(N_max), _p(score), _p(path), _p(st),
    )
    assert r == 0
    return dict(score=score, path=path, status=st)
