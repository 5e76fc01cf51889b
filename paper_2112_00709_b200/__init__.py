"""paper_2112_00709_b200 — batched log-semiring forward-backward and LF-MMI on B200.

Thin Python binding over libfb.so (include/fb.h).  Each function marshals
torch CUDA tensors to device pointers and the current CUDA stream and calls the
C-ABI entry point of the same name; every step of the path runs in the
library's sm_100a kernels.  There is no CPU fallback: a missing library or a
non-CUDA tensor raises.

    g = Graph.from_host(synth.compose(...))          # fb_graph_create
    logZ, alpha, scale, st = fb_forward(g, emis, lengths)
    post, logZb, st = fb_backward(g, emis, lengths, alpha=alpha, status=st)
    loss, totals, st = lfmmi_loss_grad(num, den, emis, lengths, grad)

Paper: arXiv 2112.00709 (PAPER.md P:173-191 log-domain recursions, P:193-227
batching, P:266-288 LF-MMI).  See DESIGN.md.
"""
from __future__ import annotations

import ctypes
from typing import Optional

import numpy as np

from ._lib import EXPORTS, lib  # noqa: F401

__all__ = [
    "FBError", "Graph", "fb_forward", "fb_backward", "fb_posteriors", "fb_gap", "lfmmi_loss_grad", "workspace_bytes",
    "fb_viterbi", "fb_forward_semiring", "fb_forward_literal", "fb_forward_backward_literal", "lfmmi_loss_grad_host", "profile_enable", "profile_reset", "profile_collect",
    "SEMIRING_LOG", "SEMIRING_TROPICAL", "SEMIRING_PROB",
    "SEQ_OK", "SEQ_EMPTY_LATTICE", "SEQ_NONFINITE_INPUT", "SEQ_BAD_LENGTH",
    "GRAPH_DEFAULT", "GRAPH_FORCE_EXACT", "GRAPH_FORCE_FACTORED", "GRAPH_CLUSTER",
]

SEQ_OK, SEQ_EMPTY_LATTICE, SEQ_NONFINITE_INPUT, SEQ_BAD_LENGTH = 0, 1, 2, 4
GRAPH_DEFAULT, GRAPH_FORCE_EXACT, GRAPH_FORCE_FACTORED, GRAPH_CLUSTER = 0, 1, 2, 4


class FBError(RuntimeError):
    def __init__(self, code: int, where: str):
        L = lib()
        msg = L.fb_status_str(code).decode()
        if code == 4:
            msg += f" ({L.fb_last_cuda_error().decode()})"
        super().__init__(f"{where}: fb_status {code}: {msg}")
        self.code = code


def _check(code: int, where: str) -> None:
    if code != 0:
        raise FBError(code, where)


def _np_ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _dev(t, dtype, name):
    """device pointer of a contiguous CUDA tensor of the given dtype (None → NULL)."""
    if t is None:
        return None
    import torch

    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def _need(cond: bool, msg: str) -> None:
    if not cond:
        raise ValueError(msg)


def _check_inputs(g: "Graph", emis, lengths, where: str):
    """Host-side shape checks the C ABI cannot make (it has no D / length arguments):
    emis is [B, N_max, g.D] and lengths has B entries; returns (B, N_max, D)."""
    _need(getattr(emis, "dim", lambda: 0)() == 3, f"{where}: emis must be [B, N_max, D]")
    B, N_max, D = emis.shape
    _need(D == g.D, f"{where}: emis has D={D} columns but the graph was built for D={g.D}")
    _need(lengths.numel() == B, f"{where}: lengths has {lengths.numel()} entries, expected B={B}")
    _need(g.G in (1, B), f"{where}: graph has G={g.G} members, expected 1 or B={B}")
    return B, N_max, D


def _check_numel(t, n: int, name: str, where: str):
    if t is not None:
        _need(t.numel() >= n, f"{where}: {name} has {t.numel()} elements, needs {n}")


def _stream():
    import torch

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class Graph:
    """A compiled fb_graph handle (G member graphs, block-diagonal)."""

    def __init__(self, state_offsets, row_ptr, col, log_w, log_init, log_final, pdf_of, D, flags=0):
        so = np.ascontiguousarray(state_offsets, np.int32)
        rp = np.ascontiguousarray(row_ptr, np.int32)
        cl = np.ascontiguousarray(col, np.int32)
        lw = np.ascontiguousarray(log_w, np.float32)
        li = np.ascontiguousarray(log_init, np.float32)
        lf = np.ascontiguousarray(log_final, np.float32)
        pd = None if pdf_of is None else np.ascontiguousarray(pdf_of, np.int32)
        h = ctypes.c_void_p()
        code = lib().fb_graph_create(ctypes.byref(h), len(so) - 1, _np_ptr(so), _np_ptr(rp), _np_ptr(cl),
                                     _np_ptr(lw), _np_ptr(li), _np_ptr(lf), _np_ptr(pd), int(D), int(flags))
        _check(code, "fb_graph_create")
        self._h = h
        self.G = len(so) - 1
        self.D = int(D)
        self.state_offsets = so
        info = np.zeros(16, np.int64)
        _check(lib().fb_graph_info(h, _np_ptr(info)), "fb_graph_info")
        keys = ["G", "K_tot", "nnz", "D", "threads", "spt", "mode", "fwd_smem", "bwd_smem", "K_max", "nnz_max",
                "fwd_slots_max", "bwd_slots_max", "U_max", "cluster_C", "cluster_S"]
        self.info = {k: int(v) for k, v in zip(keys, info)}
        self.K_tot = self.info["K_tot"]

    @classmethod
    def from_host(cls, g, flags: int = 0) -> "Graph":
        """From a synth.HostGraph (G = 1) or synth.ComposedGraph."""
        so = g.state_offsets if hasattr(g, "state_offsets") else np.array([0, g.K], np.int32)
        return cls(so, g.row_ptr, g.col, g.logw, g.log_init, g.log_final, g.pdf_of, g.D, flags)

    @property
    def handle(self):
        return self._h

    def counters(self, reset: bool = False) -> dict:
        """fb_graph_counters: exact-fallback row evaluations of the exp-factorised ⊕ (N3)."""
        out = np.zeros(2, np.int64)
        _check(lib().fb_graph_counters(self._h, _np_ptr(out), int(bool(reset))), "fb_graph_counters")
        return {"fallback_rows": int(out[0]), "fallback_rows_cluster": int(out[1])}

    def lattice_numel(self, B: int, N_max: int) -> int:
        return B * N_max * self.K_tot if self.G == 1 else N_max * self.K_tot

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().fb_graph_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def fb_forward(g: Graph, emis, lengths, alpha=None, alpha_scale=None, want_alpha=True):
    """Eq. (13).  Returns (logZ [B] f64, alpha, alpha_scale, status [B] i32)."""
    import torch

    B, N_max, D = _check_inputs(g, emis, lengths, "fb_forward")
    dev = emis.device
    _check_numel(alpha, g.lattice_numel(B, N_max), "alpha", "fb_forward")
    _check_numel(alpha_scale, B * N_max, "alpha_scale", "fb_forward")
    if want_alpha and alpha is None:
        alpha = torch.empty(g.lattice_numel(B, N_max), dtype=torch.float32, device=dev)
    if alpha is not None and alpha_scale is None:
        alpha_scale = torch.empty((B, N_max), dtype=torch.float64, device=dev)
    logZ = torch.empty(B, dtype=torch.float64, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    _check(lib().fb_forward(g.handle, _dev(emis, torch.float32, "emis"), _dev(lengths, torch.int32, "lengths"),
                            B, N_max, _dev(alpha, torch.float32, "alpha"),
                            _dev(alpha_scale, torch.float64, "alpha_scale"), _dev(logZ, torch.float64, "logZ"),
                            _dev(st, torch.int32, "status"), _stream()), "fb_forward")
    return logZ, alpha, alpha_scale, st


def fb_backward(g: Graph, emis, lengths, alpha=None, status=None, want_beta=False, post="state", post_out=None):
    """Eq. (14) (v_{n+1}) with the fused posterior epilogue (Eq. (15)).

    post: "state" (lattice layout γ), "pdf" ([B,N_max,D] Γ) or None.
    Returns (post, logZ_beta, status, beta, beta_scale)."""
    import torch

    B, N_max, D = _check_inputs(g, emis, lengths, "fb_backward")
    dev = emis.device
    if status is None:
        status = torch.zeros(B, dtype=torch.int32, device=dev)
    _check_numel(status, B, "status", "fb_backward")
    _check_numel(alpha, g.lattice_numel(B, N_max), "alpha", "fb_backward")
    beta = beta_scale = None
    if want_beta:
        beta = torch.empty(g.lattice_numel(B, N_max), dtype=torch.float32, device=dev)
        beta_scale = torch.empty((B, N_max), dtype=torch.float64, device=dev)
    pdf_level = 0
    if post is not None:
        if alpha is None:
            raise ValueError("posteriors need the forward lattice `alpha`")
        pdf_level = 1 if post == "pdf" else 0
        _check_numel(post_out, B * N_max * D if pdf_level else g.lattice_numel(B, N_max), "post_out", "fb_backward")
        if post_out is None:
            post_out = torch.empty((B, N_max, D) if pdf_level else (g.lattice_numel(B, N_max),),
                                   dtype=torch.float32, device=dev)
    logZb = torch.empty(B, dtype=torch.float64, device=dev)
    _check(lib().fb_backward(g.handle, _dev(emis, torch.float32, "emis"), _dev(lengths, torch.int32, "lengths"),
                             B, N_max, _dev(beta, torch.float32, "beta"), _dev(beta_scale, torch.float64, "beta_scale"),
                             _dev(logZb, torch.float64, "logZ_beta"), _dev(alpha, torch.float32, "alpha"),
                             _dev(post_out, torch.float32, "post"), pdf_level, _dev(status, torch.int32, "status"),
                             _stream()), "fb_backward")
    return post_out, logZb, status, beta, beta_scale


def fb_posteriors(g: Graph, alpha, beta, lengths, status, B, N_max, pdf_level=False, post=None):
    """Standalone Eq. (15): exp(α̂ + β̂ − Z_n)."""
    import torch

    dev = alpha.device
    for t, n, name in ((alpha, g.lattice_numel(B, N_max), "alpha"), (beta, g.lattice_numel(B, N_max), "beta"),
                       (lengths, B, "lengths"), (status, B, "status"),
                       (post, B * N_max * g.D if pdf_level else g.lattice_numel(B, N_max), "post")):
        _check_numel(t, n, name, "fb_posteriors")
    _need(g.G in (1, B), f"fb_posteriors: graph has G={g.G} members, expected 1 or B={B}")
    if post is None:
        post = torch.empty((B, N_max, g.D) if pdf_level else (g.lattice_numel(B, N_max),), dtype=torch.float32,
                           device=dev)
    _check(lib().fb_posteriors(g.handle, _dev(alpha, torch.float32, "alpha"), _dev(beta, torch.float32, "beta"),
                               _dev(lengths, torch.int32, "lengths"), _dev(status, torch.int32, "status"), B, N_max,
                               int(bool(pdf_level)), _dev(post, torch.float32, "post"), _stream()), "fb_posteriors")
    return post


def fb_gap(g: Graph, alpha, alpha_scale, beta, beta_scale, logZ, lengths, status=None):
    """Eq. (1) invariant diagnostic: gap[b] = max_n |⊕_k α̂_n β̂_n + C_n + D_n − logZ_b| (float64 [B])."""
    import torch

    B, N_max = alpha_scale.shape
    for t, n, name in ((alpha, g.lattice_numel(B, N_max), "alpha"), (beta, g.lattice_numel(B, N_max), "beta"),
                       (beta_scale, B * N_max, "beta_scale"), (logZ, B, "logZ"), (lengths, B, "lengths"),
                       (status, B, "status")):
        _check_numel(t, n, name, "fb_gap")
    _need(g.G in (1, B), f"fb_gap: graph has G={g.G} members, expected 1 or B={B}")
    gap = torch.empty(B, dtype=torch.float64, device=alpha.device)
    _check(lib().fb_gap(g.handle, _dev(alpha, torch.float32, "alpha"), _dev(alpha_scale, torch.float64, "alpha_scale"),
                        _dev(beta, torch.float32, "beta"), _dev(beta_scale, torch.float64, "beta_scale"),
                        _dev(logZ, torch.float64, "logZ"), _dev(lengths, torch.int32, "lengths"),
                        _dev(status, torch.int32, "status"), B, N_max, _dev(gap, torch.float64, "gap"), _stream()),
           "fb_gap")
    return gap


def workspace_bytes(num: Graph, den: Graph, B: int, N_max: int) -> int:
    return int(lib().fb_workspace_bytes(num.handle, den.handle, B, N_max))


def lfmmi_loss_grad(num: Graph, den: Graph, emis, lengths, grad=None, workspace=None, loss=None, totals=None,
                    status=None):
    """LF-MMI loss and gradient.  Returns (loss [B] f64, totals [5] f64, status [B], grad)."""
    import torch

    B, N_max, D = _check_inputs(den, emis, lengths, "lfmmi_loss_grad")
    _need(num.G == B and num.D == D, f"lfmmi_loss_grad: numerator handle has G={num.G}, D={num.D}; "
                                     f"expected G=B={B} graphs over D={D} columns")
    _need(den.G == 1, f"lfmmi_loss_grad: denominator handle has G={den.G}, expected 1")
    dev = emis.device
    for t, n, name in ((grad, B * N_max * D, "grad"), (loss, B, "loss"), (totals, 5, "totals"), (status, B, "status")):
        _check_numel(t, n, name, "lfmmi_loss_grad")
    if grad is None:
        grad = torch.empty((B, N_max, D), dtype=torch.float32, device=dev)
    nbytes = workspace_bytes(num, den, B, N_max)
    _check_numel(workspace, nbytes, "workspace", "lfmmi_loss_grad")
    if workspace is None:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    if loss is None:
        loss = torch.empty(B, dtype=torch.float64, device=dev)
    if totals is None:
        totals = torch.empty(5, dtype=torch.float64, device=dev)
    if status is None:
        status = torch.empty(B, dtype=torch.int32, device=dev)
    _check(lib().lfmmi_loss_grad(num.handle, den.handle, _dev(emis, torch.float32, "emis"),
                                 _dev(lengths, torch.int32, "lengths"), B, N_max, _dev(grad, torch.float32, "grad"),
                                 _dev(loss, torch.float64, "loss"), _dev(totals, torch.float64, "totals"),
                                 _dev(status, torch.int32, "status"), _dev(workspace, torch.uint8, "workspace"),
                                 workspace.numel(), _stream()), "lfmmi_loss_grad")
    return loss, totals, status, grad


def lfmmi_loss_grad_host(num: Graph, den: Graph, emis_host, lengths_host, bufs: dict):
    """End-to-end call with HOST inputs: pinned φ and lengths are copied to the
    device, lfmmi_loss_grad runs, and the totals (and per-utterance loss) are
    copied back.  `bufs` caches the device buffers between calls.

    Consecutive calls are pipelined: the upload of a call's φ runs on a copy
    stream into one of two device buffers while the previous call's kernels are
    still running (its buffer is reused only after the call two steps back has
    finished reading it), so a training loop is bound by max(PCIe, compute)
    rather than their sum.  Every call still uploads its own inputs and reads its
    own results back: the returned pinned tensor [Σ loss, Σ N_b, Σ logZ_num,
    Σ logZ_den, n_bad, loss_0 … loss_{B−1}] is valid after the stream synchronises
    and stays valid until the call after next (two output buffers alternate)."""
    import torch

    B, N_max, D = emis_host.shape
    dev = torch.device("cuda", torch.cuda.current_device())
    key = (B, N_max, D, dev.index, id(num), id(den))
    if bufs.get("key") not in (None, key):
        # a different batch shape or graph pair: wait for the previous calls, then reallocate
        torch.cuda.current_stream(dev).synchronize()
        bufs.clear()
    bufs["key"] = key
    if "emis" not in bufs:
        bufs["emis"] = [torch.empty((B, N_max, D), dtype=torch.float32, device=dev) for _ in range(2)]
        bufs["lengths"] = [torch.empty(B, dtype=torch.int32, device=dev) for _ in range(2)]
        bufs["grad"] = torch.empty((B, N_max, D), dtype=torch.float32, device=dev)
        bufs["ws"] = torch.empty(workspace_bytes(num, den, B, N_max), dtype=torch.uint8, device=dev)
        bufs["loss"] = torch.empty(B, dtype=torch.float64, device=dev)
        bufs["totals"] = torch.empty(5, dtype=torch.float64, device=dev)
        bufs["status"] = torch.empty(B, dtype=torch.int32, device=dev)
        bufs["out"] = [torch.empty(5 + B, dtype=torch.float64).pin_memory() for _ in range(2)]
        # two copy streams, one half of φ each: two DMA engines keep PCIe busier (measured
        # 55.5 vs 54.4 GB/s for one 512 MB copy, tools/h2d_probe.py)
        import os

        bufs["copy_streams"] = [torch.cuda.Stream(device=dev) for _ in range(int(os.environ.get("FBX_H2D_STREAMS", "2")))]
        bufs["copy_stream"] = bufs["copy_streams"][0]
        bufs["free"] = [None, None]  # event: the compute that last read buffer i has finished
        bufs["i"] = 0
    i = bufs["i"] & 1
    bufs["i"] += 1
    comp = torch.cuda.current_stream(dev)
    ncs = len(bufs["copy_streams"])
    for k, cs in enumerate(bufs["copy_streams"]):
        lo, hi = B * k // ncs, B * (k + 1) // ncs
        with torch.cuda.stream(cs):
            if bufs["free"][i] is not None:
                cs.wait_event(bufs["free"][i])
            if hi > lo:
                bufs["emis"][i][lo:hi].copy_(emis_host[lo:hi], non_blocking=True)
            if k == 0:
                bufs["lengths"][i].copy_(lengths_host, non_blocking=True)
            copied = torch.cuda.Event()
            copied.record(cs)
        comp.wait_event(copied)
    lfmmi_loss_grad(num, den, bufs["emis"][i], bufs["lengths"][i], bufs["grad"], bufs["ws"], bufs["loss"],
                    bufs["totals"], bufs["status"])
    done = torch.cuda.Event()
    done.record(comp)
    bufs["free"][i] = done
    out = bufs["out"][i]  # valid once the stream has synchronised, until the call after next
    out[:5].copy_(bufs["totals"], non_blocking=True)
    out[5:].copy_(bufs["loss"], non_blocking=True)
    return out


def fb_viterbi(g: Graph, emis, lengths):
    """Tropical-semiring best path.  Returns (score [B] f64, path [B,N_max] i32, status)."""
    import torch

    B, N_max, D = _check_inputs(g, emis, lengths, "fb_viterbi")
    dev = emis.device
    nbytes = int(lib().fb_viterbi_workspace_bytes(g.handle, B, N_max))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    score = torch.empty(B, dtype=torch.float64, device=dev)
    path = torch.empty((B, N_max), dtype=torch.int32, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    _check(lib().fb_viterbi(g.handle, _dev(emis, torch.float32, "emis"), _dev(lengths, torch.int32, "lengths"), B,
                            N_max, _dev(score, torch.float64, "score"), _dev(path, torch.int32, "path"),
                            _dev(st, torch.int32, "status"), _dev(ws, torch.uint8, "workspace"), ws.numel(),
                            _stream()), "fb_viterbi")
    return score, path, st


SEMIRING_LOG, SEMIRING_TROPICAL, SEMIRING_PROB = 0, 1, 2


def fb_forward_literal(g: Graph, emis, lengths, semiring: int = SEMIRING_LOG):
    """The paper's literal strategy (N4): one block-diagonal batch SpMV per frame with
    phony-state padding, in the log / tropical / probability semiring.  Returns score [B] f64."""
    import torch

    B, N_max, D = _check_inputs(g, emis, lengths, "fb_forward_literal")
    dev = emis.device
    nbytes = int(lib().fb_literal_workspace_bytes(g.handle, B))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    score = torch.empty(B, dtype=torch.float64, device=dev)
    _check(lib().fb_forward_literal(g.handle, int(semiring), _dev(emis, torch.float32, "emis"),
                                    _dev(lengths, torch.int32, "lengths"), B, N_max,
                                    _dev(score, torch.float64, "score"), _dev(ws, torch.uint8, "workspace"),
                                    ws.numel(), _stream()), "fb_forward_literal")
    return score


def fb_forward_semiring(g: Graph, emis, lengths, semiring: int = SEMIRING_LOG):
    """The fused forward (Eq. (13)) in the log / tropical / probability semiring (N4).
    Returns (score [B] f64, status [B] i32)."""
    import torch

    B, N_max, D = _check_inputs(g, emis, lengths, "fb_forward_semiring")
    dev = emis.device
    score = torch.empty(B, dtype=torch.float64, device=dev)
    st = torch.empty(B, dtype=torch.int32, device=dev)
    _check(lib().fb_forward_semiring(g.handle, int(semiring), _dev(emis, torch.float32, "emis"),
                                     _dev(lengths, torch.int32, "lengths"), B, N_max, _dev(score, torch.float64, "score"),
                                     _dev(st, torch.int32, "status"), _stream()), "fb_forward_semiring")
    return score, st


def fb_forward_backward_literal(g: Graph, emis, lengths, semiring: int = SEMIRING_LOG, want_post: bool = True):
    """The literal strategy's forward-backward (N4): one batch SpMV per frame in each
    direction, posteriors X ⊗ y ⊘ Z in the semiring.  Returns (score [B] f64, post f64
    in the lattice layout, or None)."""
    import torch

    B, N_max, D = _check_inputs(g, emis, lengths, "fb_forward_backward_literal")
    dev = emis.device
    nbytes = int(lib().fb_literal_fb_workspace_bytes(g.handle, B, N_max))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)
    score = torch.empty(B, dtype=torch.float64, device=dev)
    post = torch.empty(g.lattice_numel(B, N_max), dtype=torch.float64, device=dev) if want_post else None
    _check(lib().fb_forward_backward_literal(g.handle, int(semiring), _dev(emis, torch.float32, "emis"),
                                             _dev(lengths, torch.int32, "lengths"), B, N_max,
                                             _dev(score, torch.float64, "score"), _dev(post, torch.float64, "post"),
                                             _dev(ws, torch.uint8, "workspace"), ws.numel(), _stream()),
           "fb_forward_backward_literal")
    return score, post


def profile_enable(on: bool = True) -> None:
    lib().fb_profile_enable(1 if on else 0)


def profile_reset() -> None:
    lib().fb_profile_reset()


def profile_collect() -> dict:
    """{kernel name: (launches, summed device ms)} since the last reset."""
    cap = 32
    names = (ctypes.c_char_p * cap)()
    counts = np.zeros(cap, np.int64)
    ms = np.zeros(cap, np.float64)
    n = ctypes.c_int32(0)
    _check(lib().fb_profile_collect(names, _np_ptr(counts), _np_ptr(ms), cap, ctypes.byref(n)), "fb_profile_collect")
    return {names[i].decode(): (int(counts[i]), float(ms[i])) for i in range(n.value)}
