"""In-step kernel timing under different host loads (diagnostic, not a bench line).

The bench's in-step GEMM event pairs (roofline.achieved) read ~8 % slower than the
same launches under ncu or in the back-to-back probe. This runs a C2-width engine at
reduced depth with the bench's options and varies only the host side:

  bench     the bench's options (host Adam overlapped, optimizer team pinned, 15/16 CPUs)
  skip_opt  no host Adam at all (the GPU work and transfers are unchanged)
  team8     host Adam on an 8-thread team (half the CPUs idle)

and prints CUDA-event ms per GEMM / attention launch for each, so host contention on
the thread that issues the compute stream can be told apart from on-GPU effects.

  python tools/instep_probe.py [layers=4] [steps=4]
"""
import ctypes
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2602_04816_b200 import engine as E  # noqa: E402
from paper_2602_04816_b200 import _lib  # noqa: E402


def kt(lib, kind):
    ms, w, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
    lib.hlm_ktimer_collect(kind, ctypes.byref(ms), ctypes.byref(w), ctypes.byref(n))
    return ms.value, w.value, n.value


class Nvml:
    """SM clock and board power sampled every 2 ms on a side thread (NVML)."""

    def __init__(self):
        import pynvml
        pynvml.nvmlInit()
        self.nv = pynvml
        self.h = pynvml.nvmlDeviceGetHandleByIndex(0)
        self.clk, self.pw, self.stop_ = [], [], False

    def _loop(self):
        while not self.stop_:
            self.clk.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.pw.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1e3)
            time.sleep(0.002)

    def start(self):
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()

    def stop(self):
        self.stop_ = True
        self.t.join()
        c, p = np.array(self.clk), np.array(self.pw)
        return {"sm_mhz_median": float(np.median(c)), "sm_mhz_p10": float(np.percentile(c, 10)),
                "share_below_1900": float((c < 1900).mean()), "power_w_mean": float(p.mean()),
                "power_w_max": float(p.max()), "samples": int(len(c))}


def run(variant, layers, steps, warmup=2):
    lib = _lib.lib()
    cfg = E.ModelConfig(layers, 3584, 18944, 152064, 2048, 8, k_ckpt=1, n_heads=28, rope_theta=1e6)
    store = E.Store(cfg, 1234, "bf16", init="parallel")
    arena = E.Arena(cfg, device=0, weight_cache_bytes=layers * (2 * cfg.block_params() + 256))
    opts = dict(eager_optim=True, threaded_accum=True, n_slab=layers + 4, grad_buffers=8,
                sparse_embed_grad=True, embed_gather_host=True, pin_threads=True, record_trace=True,
                overlap_optimizer_tail=True, tail_blocks=layers)
    if variant == "skip_opt":
        opts.update(skip_optimizer=True, overlap_optimizer_tail=False, eager_optim=False)
    if variant == "team8":
        opts.update(host_threads=8)
    eng = E.Engine(store, arena, E.HyperParams(lr=1e-4), E.EngineOptions(**opts))
    batches = [E.make_copy_task_batch(cfg, 1235, skip=i) for i in range(warmup + steps)]
    for i in range(warmup):
        eng.train_step(batches[i])
    eng.wait_optimizer()
    lib.hlm_ktimer_reset()
    lib.hlm_ktimer_enable(1)
    nv = Nvml()
    nv.start()
    t0 = time.perf_counter()
    for i in range(steps):
        eng.train_step(batches[warmup + i])
    eng.wait_optimizer()
    wall = time.perf_counter() - t0
    clocks = nv.stop()
    lib.hlm_ktimer_enable(0)
    out = {"variant": variant, "layers": layers, "s_per_step": wall / steps, "clocks": clocks}
    for kind, name in ((0, "gemm"), (1, "attn_fwd"), (2, "attn_bwd"), (4, "rmsnorm_bwd")):
        ms, w, n = kt(lib, kind)
        out[name] = {"ms_per_launch": ms / max(1, n), "launches": n,
                     "rate": w / (ms / 1e3) / (1e12 if kind < 3 else 1e9) if ms > 0 else None}
    lib.hlm_ktimer_reset()
    del eng, arena, store
    return out


if __name__ == "__main__":
    layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    for v in (sys.argv[3].split(",") if len(sys.argv) > 3 else ["bench", "skip_opt", "team8", "bench"]):
        print(json.dumps(run(v, layers, steps)), flush=True)
