"""Run the block-GEMM roofline probe once (used under ncu)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_04816_b200 import _lib
L = _lib.blib()
L.hlm_cuda_bench_block_gemms.argtypes = [ctypes.POINTER(_lib.HlmBlockDims), ctypes.c_int] + [ctypes.POINTER(ctypes.c_double)] * 3
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
dims = {"c2": (8, 2048, 3584, 18944, 28)}[cfg]
d = _lib.HlmBlockDims(*dims, 0)
fl, ms, ml = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
_lib.check(L.hlm_cuda_bench_block_gemms(ctypes.byref(d), int(sys.argv[2]) if len(sys.argv) > 2 else 5, ctypes.byref(fl), ctypes.byref(ms), ctypes.byref(ml)))
print(f"block GEMM set: {fl.value/1e12:.2f} TFLOP in {ms.value:.3f} ms -> {fl.value/ms.value/1e9:.1f} TFLOP/s; {ml.value:.3f} ms/launch")
