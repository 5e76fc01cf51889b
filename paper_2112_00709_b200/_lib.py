"""ctypes loader for libfb.so (the C-ABI of include/fb.h).  No fallback: if the
library is missing or cannot be loaded the import of any compute entry point
raises."""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FBX_LIB") or os.path.join(_HERE, "libfb.so")  # FBX_LIB: A/B experiments
_lock = threading.Lock()
_lib = None

c_i32 = ctypes.c_int32
c_i64 = ctypes.c_int64
c_p = ctypes.c_void_p
c_sz = ctypes.c_size_t

_SIGS = {
    "fb_graph_create": (c_i32, [ctypes.POINTER(c_p), c_i32, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_i32, c_i32]),
    "fb_graph_destroy": (c_i32, [c_p]),
    "fb_graph_info": (c_i32, [c_p, c_p]),
    "fb_graph_counters": (c_i32, [c_p, c_p, c_i32]),
    "fb_forward": (c_i32, [c_p, c_p, c_p, c_i32, c_i32, c_p, c_p, c_p, c_p, c_p]),
    "fb_backward": (c_i32, [c_p, c_p, c_p, c_i32, c_i32, c_p, c_p, c_p, c_p, c_p, c_i32, c_p, c_p]),
    "fb_posteriors": (c_i32, [c_p, c_p, c_p, c_p, c_p, c_i32, c_i32, c_i32, c_p, c_p]),
    "fb_gap": (c_i32, [c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_p, c_i32, c_i32, c_p, c_p]),
    "fb_workspace_bytes": (c_sz, [c_p, c_p, c_i32, c_i32]),
    "lfmmi_loss_grad": (c_i32, [c_p, c_p, c_p, c_p, c_i32, c_i32, c_p, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "fb_viterbi_workspace_bytes": (c_sz, [c_p, c_i32, c_i32]),
    "fb_viterbi": (c_i32, [c_p, c_p, c_p, c_i32, c_i32, c_p, c_p, c_p, c_p, c_sz, c_p]),
    "fb_literal_workspace_bytes": (c_sz, [c_p, c_i32]),
    "fb_forward_literal": (c_i32, [c_p, c_i32, c_p, c_p, c_i32, c_i32, c_p, c_p, c_sz, c_p]),
    "fb_forward_semiring": (c_i32, [c_p, c_i32, c_p, c_p, c_i32, c_i32, c_p, c_p, c_p]),
    "fb_literal_fb_workspace_bytes": (c_sz, [c_p, c_i32, c_i32]),
    "fb_forward_backward_literal": (c_i32, [c_p, c_i32, c_p, c_p, c_i32, c_i32, c_p, c_p, c_p, c_sz, c_p]),
    "fb_profile_enable": (None, [c_i32]),
    "fb_profile_reset": (None, []),
    "fb_profile_collect": (c_i32, [c_p, c_p, c_p, c_i32, c_p]),
    "fb_status_str": (ctypes.c_char_p, [c_i32]),
    "fb_last_cuda_error": (ctypes.c_char_p, []),
}

EXPORTS = tuple(_SIGS)


def lib():
    """Load libfb.so once (raises if it is missing: there is no CPU fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RuntimeError(
                    f"{LIB_PATH} is not built; run `python -m paper_2112_00709_b200.build` "
                    "(the CUDA library is the only implementation)")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in _SIGS.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            _lib = L
    return _lib
