"""Achieved HBM GB/s of the block's elementwise / norm kernels (hlm_cuda_bench_block_ops)."""
import ctypes, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_04816_b200 import _lib
L = _lib.blib()
shapes = {"c2": (8, 2048, 3584, 18944, 28), "c5": (1, 4096, 12288, 49152, 96), "c1": (4, 128, 256, 1024, 2)}
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
d = _lib.HlmBlockDims(*shapes[cfg], 0)
gbs, ms = (ctypes.c_double * 6)(), (ctypes.c_double * 6)()
_lib.check(L.hlm_cuda_bench_block_ops(ctypes.byref(d), 20, gbs, ms))
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
for i, k in enumerate(("rmsnorm_fwd", "rmsnorm_bwd", "swiglu_fwd", "swiglu_bwd", "rope", "cast_bf16")):
    print(f"{cfg} {k:12s} {ms[i]*1e3:8.1f} us  {gbs[i]:7.0f} GB/s  {gbs[i]/peak:5.2f} of HBM")
