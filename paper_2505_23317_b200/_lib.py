"""ctypes declarations of libcfdetr.so (include/cfdetr.h, include/cfdetr_debug.h).

Argument marshalling only.  Loading fails loudly if the library is missing: there
is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CFD_LIB_DEBUG=1: the debug / trace build; CFD_LIB_VARIANT=name: libcfdetr_<name>.so (A/B timing builds)
LIB_PATH = os.path.join(HERE, "libcfdetr_dbg.so" if os.environ.get("CFD_LIB_DEBUG") == "1" else
                        f"libcfdetr_{os.environ['CFD_LIB_VARIANT']}.so" if os.environ.get("CFD_LIB_VARIANT") else
                        "libcfdetr.so")

P = C.c_void_p
I32 = C.c_int32
I64 = C.c_int64
F32 = C.c_float
SZ = C.c_size_t

STATUS = {0: "CFD_OK", -1: "CFD_E_ARG", -2: "CFD_E_SHAPE", -3: "CFD_E_UNSUPPORTED", -4: "CFD_E_CAPACITY",
          -5: "CFD_E_CUDA", -6: "CFD_E_DEVICE"}

# public symbols of include/cfdetr.h and include/cfdetr_debug.h
PUBLIC_SYMBOLS = ["cfd_create", "cfd_destroy", "cfd_query", "cfd_coarse_encode", "cfd_select_regions",
                  "cfd_refine_encode", "cfd_batch_refine", "cfd_batch_refine_padded", "cfd_check", "cfd_status_str", "cfd_version",
                  "cfd_hardness", "cfd_box_scores", "cfd_set_decoder", "cfd_decode", "cfd_frames_from_u8"]
DEBUG_SYMBOLS = ["cfdx_gemm", "cfdx_gemm_resid_ln", "cfdx_attention", "cfdx_layernorm", "cfdx_score", "cfdx_gather",
                 "cfdx_launch_count", "cfdx_mlp_trace", "cfdx_attn_trace", "cfdx_probe_install", "cfdx_probe_count", "cfdx_set_option",
                 "cfdx_frames_u8"]
PROBE_KINDS = {"attention": 0, "score": 1, "gemm_qkv": 2, "gemm_oproj": 3, "gemm_mlp1": 4, "gemm_mlp2": 5,
               "gemm_embed_c": 6, "gemm_embed_f": 7, "layernorm": 8, "select": 9, "gather": 10, "im2col": 11,
               "meta": 12}


class cfd_config(C.Structure):
    _fields_ = [("img_h", I32), ("img_w", I32), ("patch_coarse", I32), ("patch_fine", I32), ("d_model", I32),
                ("n_heads", I32), ("n_layers", I32), ("d_ff", I32), ("score_layer", I32), ("max_tasks", I32),
                ("ln_eps", F32)]


class cfd_layer_weights(C.Structure):
    _fields_ = [("w_qkv", P), ("w_o", P), ("w_1", P), ("w_2", P), ("b_qkv", P), ("b_o", P), ("b_1", P),
                ("b_2", P), ("ln1_g", P), ("ln1_b", P), ("ln2_g", P), ("ln2_b", P)]


class cfd_weights(C.Structure):
    _fields_ = [("w_embed_c", P), ("w_embed_f", P), ("b_embed_c", P), ("b_embed_f", P), ("pe_c", P),
                ("pe_f", P), ("h_layers", C.POINTER(cfd_layer_weights))]


class cfd_decoder_weights(C.Structure):
    _fields_ = [("n_queries", I32), ("queries", P), ("ln_q_g", P), ("ln_q_b", P), ("ln_m_g", P), ("ln_m_b", P),
                ("w_q", P), ("w_kv", P), ("w_o", P), ("b_q", P), ("b_kv", P), ("b_o", P), ("w_head", P),
                ("b_head", P)]


class CfdError(RuntimeError):
    def __init__(self, fn: str, status: int):
        super().__init__(f"{fn} failed: {STATUS.get(status, status)}")
        self.status = status


_lib = None


def load() -> C.CDLL:
    """Load libcfdetr.so (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2505_23317_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    sig = {
        "cfd_create": [C.POINTER(cfd_config), C.POINTER(cfd_weights), P, C.POINTER(P)],
        "cfd_destroy": [P],
        "cfd_query": [P, I32, C.POINTER(I32), C.POINTER(I32), C.POINTER(I32), C.POINTER(SZ)],
        "cfd_coarse_encode": [P, I32, P, P, P, P, P, P, SZ, P],
        "cfd_select_regions": [P, I32, P, I32, C.POINTER(I32), F32, P, P, P],
        "cfd_refine_encode": [P, P, P, P, P, P, P, P, P, P, SZ, P],
        "cfd_batch_refine": [P, I32, P, P, P, P, C.POINTER(I32), P, P, P, P, P, SZ, P],
        "cfd_batch_refine_padded": [P, I32, P, P, P, P, I32, P, P, P, P, P, P, SZ, P],
        "cfd_check": [P, P],
        "cfd_hardness": [P, I32, I32, P, F32, F32, P, P],
        "cfd_box_scores": [P, I32, I32, P, P, F32, F32, P, P],
        "cfd_set_decoder": [P, C.POINTER(cfd_decoder_weights), P],
        "cfd_decode": [P, I32, P, P, I32, P, P, P, P, SZ, P],
        "cfd_frames_from_u8": [P, I32, P, C.POINTER(F32), C.POINTER(F32), P, P],
        "cfdx_frames_u8": [I64, P, C.POINTER(F32), C.POINTER(F32), P, P],
        "cfd_status_str": [I32],
        "cfd_version": [],
        "cfdx_gemm": [I32, I32, I32, P, P, P, I32, P, P, P],
        "cfdx_gemm_resid_ln": [I32, I32, I32, P, P, P, P, P, P, F32, P, I32, I32, P],
        "cfdx_attention": [I32, P, I32, I32, I32, I32, P, P, P, I32, P, P],
        "cfdx_layernorm": [I32, I32, P, P, P, F32, P, P],
        "cfdx_score": [I32, I32, I32, I32, P, I32, P, I32, P, P],
        "cfdx_gather": [P, I32, P, P, P, P, P, P, P, P, P, P, P, P],
        "cfdx_launch_count": [],
        "cfdx_mlp_trace": [P, I32],
        "cfdx_attn_trace": [P, I32],
        "cfdx_probe_install": [I32, C.POINTER(P), C.POINTER(P), I32],
        "cfdx_probe_count": [I32],
        "cfdx_set_option": [P, I32, I32],
    }
    for name, args in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = I32
    lib.cfd_status_str.restype = C.c_char_p
    lib.cfd_version.restype = C.c_char_p
    lib.cfdx_launch_count.restype = I64
    _lib = lib
    return lib


def check(fn: str, status: int) -> None:
    if status != 0:
        raise CfdError(fn, status)
