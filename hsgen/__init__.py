"""Seeded synthetic inputs shared by the oracle (tests) and the CUDA path (bench).

Thin ctypes wrapper over ``libhsgen.so`` (``hsgen/hsgen.c``).  Holds no arithmetic of the
method: random draws, the model shapes of the paper's workloads, and the host-image writer
(byte layout documented in ``include/hs.h``).

Shapes: Llama-2 7B / 13B (the paper's models,
PAPER.md:817, sizes 12.5 GB / 24.2 GB in PAPER.md:754-755) and a tiny decoder (BASELINE
config 1).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
_SO = os.path.join(_HERE, "libhsgen.so")

HS_MAX_LAYERS = 128
HEADER_BYTES = 65536


class ModelCfg(C.Structure):
    _fields_ = [("n_layers", C.c_int32), ("hidden", C.c_int32), ("n_heads", C.c_int32),
                ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32),
                ("vocab", C.c_int32), ("max_seq", C.c_int32), ("rms_eps", C.c_float),
                ("rope_theta", C.c_float)]


class ImageHeader(C.Structure):
    _fields_ = [("magic", C.c_uint64), ("version", C.c_uint32), ("gu_interleave", C.c_uint32),
                ("cfg", ModelCfg), ("total_bytes", C.c_uint64), ("embed_off", C.c_uint64),
                ("embed_bytes", C.c_uint64), ("layer_off", C.c_uint64 * HS_MAX_LAYERS),
                ("layer_bytes", C.c_uint64), ("t_attn_norm", C.c_uint64), ("t_wqkv", C.c_uint64),
                ("t_wo", C.c_uint64), ("t_ffn_norm", C.c_uint64), ("t_wgu", C.c_uint64),
                ("t_wd", C.c_uint64), ("final_off", C.c_uint64), ("final_bytes", C.c_uint64),
                ("t_final_norm", C.c_uint64), ("t_lm_head", C.c_uint64), ("param_bytes", C.c_uint64)]


def _make_cfg(n_layers, hidden, n_heads, head_dim, ffn, vocab, max_seq=4096):
    return dict(n_layers=n_layers, hidden=hidden, n_heads=n_heads, n_kv_heads=n_heads,
                head_dim=head_dim, ffn=ffn, vocab=vocab, max_seq=max_seq, rms_eps=1e-5,
                rope_theta=10000.0)


# Model shapes.  Llama-2 (7B: L32 H4096 32x128 F11008 V32000; 13B: L40 H5120 40x128 F13824)
CONFIGS = {
    "tiny": _make_cfg(4, 256, 4, 64, 768, 1024, 1024),
    "llama2-7b": _make_cfg(32, 4096, 32, 128, 11008, 32000),
    "llama2-13b": _make_cfg(40, 5120, 40, 128, 13824, 32000),
}

WEIGHT_SEED = 1234  # weight seed 1234, prompt seed 42 + request index
PROMPT_SEED = 42

# tensor ids (include/hsgen.h)
EMBED, FINAL_NORM, LM_HEAD = 0, 1, 2
ATTN_NORM, WQ, WK, WV, WO, FFN_NORM, WG, WU, WD = range(9)


def layer_tensor(layer: int, k: int) -> int:
    return 16 + 16 * layer + k


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "hsgen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-fPIC", "-shared", "-fopenmp",
                               "-I" + os.path.join(_ROOT, "include"), src, "-o", _SO, "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        L.hsgen_tensor_spec.argtypes = [C.POINTER(ModelCfg), C.c_uint32, C.POINTER(C.c_int64),
                                        C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.hsgen_tensor_bf16.argtypes = [C.POINTER(ModelCfg), C.c_uint64, C.c_uint32, C.c_uint64,
                                        C.c_uint64, C.c_void_p, C.c_int32]
        L.hsgen_tensor_bf16.restype = None
        L.hsgen_normal.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64]
        L.hsgen_normal.restype = C.c_double
        L.hsgen_image_layout.argtypes = [C.POINTER(ModelCfg), C.POINTER(ImageHeader)]
        L.hsgen_image_layout.restype = C.c_uint64
        L.hsgen_image_fill.argtypes = [C.POINTER(ImageHeader), C.c_uint64, C.c_void_p, C.c_uint64,
                                       C.c_uint64, C.c_int32]
        L.hsgen_tokens.argtypes = [C.c_uint64, C.c_int64, C.c_int32, C.c_void_p]
        L.hsgen_tokens.restype = None
        _lib = L
    return _lib


def cfg_struct(cfg: dict) -> ModelCfg:
    return ModelCfg(**cfg)


def tensor_spec(cfg: dict, tensor_id: int):
    r, c, s, o = C.c_int64(), C.c_int64(), C.c_double(), C.c_double()
    c_cfg = cfg_struct(cfg)
    if lib().hsgen_tensor_spec(C.byref(c_cfg), tensor_id, C.byref(r), C.byref(c), C.byref(s), C.byref(o)) != 0:
        raise KeyError(tensor_id)
    return r.value, c.value, s.value, o.value


def tensor_bf16(cfg: dict, seed: int, tensor_id: int, nthreads: int = 0) -> np.ndarray:
    """Logical tensor (rows x cols) as bf16 bit patterns (uint16)."""
    rows, cols, _, _ = tensor_spec(cfg, tensor_id)
    out = np.empty((rows, cols), dtype=np.uint16)
    c_cfg = cfg_struct(cfg)
    lib().hsgen_tensor_bf16(C.byref(c_cfg), seed, tensor_id, 0, rows * cols,
                            out.ctypes.data, nthreads)
    return out


def normal(seed: int, tensor_id: int, index: int) -> float:
    return lib().hsgen_normal(seed, tensor_id, index)


def image_header(cfg: dict) -> ImageHeader:
    h = ImageHeader()
    c_cfg = cfg_struct(cfg)
    if lib().hsgen_image_layout(C.byref(c_cfg), C.byref(h)) == 0:
        raise ValueError("invalid model cfg")
    return h


def image_fill(header: ImageHeader, seed: int, dst_ptr: int, begin: int, end: int,
               nthreads: int = 0) -> None:
    """Write image bytes [begin, end) to raw host address dst_ptr."""
    if lib().hsgen_image_fill(C.byref(header), seed, C.c_void_p(dst_ptr), begin, end, nthreads) != 0:
        raise ValueError("image_fill failed")


def image_bytes(cfg: dict, seed: int = WEIGHT_SEED, begin: int = 0, end: int | None = None) -> np.ndarray:
    """Image bytes [begin, end) as a numpy uint8 array (small models / tests)."""
    h = image_header(cfg)
    end = h.total_bytes if end is None else end
    buf = np.empty(end - begin, dtype=np.uint8)
    image_fill(h, seed, buf.ctypes.data, begin, end)
    return buf


def tokens(seed: int, n: int, vocab: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int32)
    lib().hsgen_tokens(seed, n, vocab, out.ctypes.data)
    return out


def prompts(n_seqs: int, length: int, vocab: int, seed0: int = PROMPT_SEED):
    """Prompts of request i drawn from stream seed0 + i."""
    return [tokens(seed0 + i, length, vocab) for i in range(n_seqs)]
