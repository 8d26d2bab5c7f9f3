"""ctypes binding of the C ABI declared in include/hlm_cuda.h.

The shared library is built in-tree (``paper_2602_04816_b200/libhlm_b200.so``)
by ``__graft_entry__.build()``; loading fails loudly when it is missing — there
is no CPU fallback for any GPU stage.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# HLM_LIB_PATH: an alternative build of the same library (A/B timing tools only)
LIB_PATH = os.environ.get("HLM_LIB_PATH") or os.path.join(_HERE, "libhlm_b200.so")

_lib = None


class HlmError(RuntimeError):
    """Non-zero status from the C ABI; ``code`` is the HlmStatus value."""

    def __init__(self, code, msg):
        super().__init__(f"[hlm status {code}] {msg}")
        self.code = code


class HlmGemmDesc(ctypes.Structure):
    _fields_ = [
        ("M", ctypes.c_int), ("N", ctypes.c_int), ("K", ctypes.c_int), ("G", ctypes.c_int),
        ("kgroup", ctypes.c_int),
        ("a_mn", ctypes.c_int), ("b_mn", ctypes.c_int),
        ("a_grouped", ctypes.c_int), ("b_grouped", ctypes.c_int),
        ("epi", ctypes.c_int),
        ("A", ctypes.c_void_p), ("lda", ctypes.c_longlong), ("a_gstride", ctypes.c_longlong),
        ("B", ctypes.c_void_p), ("ldb", ctypes.c_longlong), ("b_gstride", ctypes.c_longlong),
        ("C", ctypes.c_void_p), ("ldc", ctypes.c_longlong), ("c_gstride", ctypes.c_longlong),
        ("R", ctypes.c_void_p), ("ldr", ctypes.c_longlong), ("r_gstride", ctypes.c_longlong),
        ("rope_cos", ctypes.c_void_p), ("rope_sin", ctypes.c_void_p),
        ("rope_seq", ctypes.c_int), ("rope_head_dim", ctypes.c_int),
        ("aux", ctypes.c_void_p), ("aux_ld", ctypes.c_longlong), ("aux_gstride", ctypes.c_longlong),
        ("C2", ctypes.c_void_p), ("ldc2", ctypes.c_longlong),
    ]


EPI_BF16, EPI_F32, EPI_F32_ADD, EPI_BF16_ROPE, EPI_SWIGLU, EPI_SWIGLU_BWD = 0, 1, 2, 3, 4, 5


def lib():
    """Load libhlm_b200.so once; raise if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: run __graft_entry__.build() (make -C "
                "paper_2602_04816_b200/csrc). The CUDA path has no fallback.")
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.hlm_cuda_last_error.restype = ctypes.c_char_p
        _lib.hlm_cuda_gemm.argtypes = [ctypes.POINTER(HlmGemmDesc), ctypes.c_void_p]
    return _lib


def check(rc):
    if rc != 0:
        raise HlmError(rc, lib().hlm_cuda_last_error().decode())
    return rc


def gemm(desc, stream=0):
    check(lib().hlm_cuda_gemm(ctypes.byref(desc), ctypes.c_void_p(stream)))


class HlmBlockDims(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("seq", ctypes.c_int64), ("hidden", ctypes.c_int64),
                ("ffn", ctypes.c_int64), ("n_heads", ctypes.c_int32), ("flags", ctypes.c_int32)]


BLOCK_GENERIC_ATTENTION = 1
BLOCK_UNFUSED = 2
_vp = ctypes.c_void_p


def _setup_block_protos(L):
    L.hlm_cuda_block_acts_bytes.restype = ctypes.c_size_t
    L.hlm_cuda_block_acts_bytes.argtypes = [ctypes.POINTER(HlmBlockDims)]
    L.hlm_cuda_block_ws_bytes.restype = ctypes.c_size_t
    L.hlm_cuda_block_ws_bytes.argtypes = [ctypes.POINTER(HlmBlockDims)]
    L.hlm_cuda_block_fwd.argtypes = [ctypes.POINTER(HlmBlockDims)] + [_vp] * 8
    L.hlm_cuda_block_bwd.argtypes = [ctypes.POINTER(HlmBlockDims)] + [_vp] * 10
    L.hlm_cuda_rope_table.argtypes = [_vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_double]
    L.hlm_cuda_head_ws_bytes.restype = ctypes.c_size_t
    L.hlm_cuda_head_ws_bytes.argtypes = [ctypes.c_int64] * 3
    L.hlm_cuda_head_loss.argtypes = [ctypes.c_int64] * 3 + [_vp, _vp, _vp, ctypes.c_float, _vp, _vp,
                                                            ctypes.c_int, _vp, _vp, _vp]
    L.hlm_cuda_head_stats.argtypes = [ctypes.c_int64] * 3 + [_vp, _vp, _vp, ctypes.c_float, _vp, _vp, _vp,
                                                             _vp]
    L.hlm_cuda_head_grad_chunk.argtypes = [ctypes.c_int64] * 3 + [_vp, _vp, ctypes.c_float, ctypes.c_int64,
                                                                  ctypes.c_int64, _vp, ctypes.c_int, _vp,
                                                                  ctypes.c_int, _vp, _vp]
    L.hlm_cuda_head_chunk_vocab.restype = ctypes.c_int64
    L.hlm_cuda_head_chunk_vocab.argtypes = [ctypes.c_int64] * 2
    L.hlm_cuda_embed_fwd.argtypes = [_vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                     _vp, _vp]
    L.hlm_cuda_embed_bwd.argtypes = [_vp, _vp, _vp, _vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                     _vp]
    L.hlm_embed_csr.argtypes = [_vp, ctypes.c_int64, ctypes.c_int64, _vp, _vp]
    L.hlm_cuda_cast_bf16.argtypes = [_vp, _vp, ctypes.c_int64, _vp]
    L.hlm_cuda_attention_fwd.argtypes = [ctypes.POINTER(HlmBlockDims)] + [_vp] * 5 + [ctypes.c_int64, _vp]
    L.hlm_cuda_attention_bwd.argtypes = [ctypes.POINTER(HlmBlockDims)] + [_vp] * 10 + [ctypes.c_int64,
                                                                                         _vp]


_block_ready = False


def blib():
    global _block_ready
    L = lib()
    if not _block_ready:
        _setup_block_protos(L)
        _block_ready = True
    return L
