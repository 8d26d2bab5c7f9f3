#!/usr/bin/env python
"""Benchmark of the layer-streaming training step (BASELINE.json metric:
train tokens/s & TFLOPS; H2D GB/s and overlap vs roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c2]

Workload (N=1 default): BASELINE.json configs[1], the Qwen2.5-7B-shaped
decoder — L28 h3584 f18944 V152064 S2048 B8 (T = 16384 tokens), 28 heads of
128, RoPE theta 1e6, untied, K_ckpt = 1 — host-resident FP32 master + Adam
(115 GB) with BF16 layer streaming, on 1 B200. One step = one full training
step (forward, loss, recompute + backward, FP32 gradient D2H, host Adam on
every parameter). Synthetic copy-task tokens, random-init weights.

--impl reference times the reference's own CPU implementation of the same
step (oracle/_ref, the reference library compiled from its sources) on a
bounded sample: one block fwd + recompute + bwd and the head at full width on
T = 4 tokens, extrapolated linearly in T and L (labelled an estimate).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c1": dict(layers=4, hidden=256, ffn=1024, vocab=1024, seq=128, batch=4, n_heads=2),
    "c2": dict(layers=28, hidden=3584, ffn=18944, vocab=152064, seq=2048, batch=8, n_heads=28),
    "c3": dict(layers=64, hidden=5120, ffn=27648, vocab=152064, seq=2048, batch=8, n_heads=40),
    "c4": dict(layers=80, hidden=8192, ffn=29568, vocab=152064, seq=2048, batch=8, n_heads=64),
    "c5": dict(layers=48, hidden=12288, ffn=49152, vocab=201088, seq=4096, batch=8, n_heads=96),
}
NAMES = {"c1": "tiny-qwen-style-L4-d256-s128", "c2": "qwen2.5-7b-shaped-L28-d3584-s2048",
         "c3": "qwen2.5-32b-shaped-L64-d5120-s2048", "c4": "qwen2.5-72b-shaped-L80-d8192-s2048",
         "c5": "dense-120b-class-L48-d12288-s4096"}
METRIC = "train_tokens_per_s"
PCIE_ASSUMED_GBS = 55.0   # measured on the pool's box: pinned H2D 55.5 / D2H 55.8 GB/s



def _mem_available():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return None


def pick_slabs(args, m, nums, world, local_world):
    """Gradient slab count and optimizer tail. The host never idles while a
    gradient is in flight, so the pool should hold a whole step's backlog of
    block gradients (layers + 4 slabs: two widest-tile slabs for the embedding /
    head, the rest block-sized), capped by the host memory left after the
    store (16 GB reserve); the tail then covers every block."""
    n_slab = args.slabs
    if n_slab <= 0:
        block = 4 * nums["n"] // world
        wide = 4 * m["vocab"] * m["hidden"] // world
        avail = _mem_available()
        n_slab = m["layers"] + 4
        if avail is not None:
            budget = (avail - 16e9) / max(1, local_world) - 2 * max(wide, block)
            n_slab = min(n_slab, 2 + int(budget // block))
        n_slab = max(6, n_slab)
    tail = args.tail_blocks
    if tail == -2:
        tail = min(m["layers"], n_slab - 3)
    return n_slab, tail

def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d["hbm_gbs"], d["bf16_tflops"], d["bf16_tflops_sustained"], "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


def model_numbers(m):
    L, h, f, V, S, B = m["layers"], m["hidden"], m["ffn"], m["vocab"], m["seq"], m["batch"]
    T = B * S
    n_mm = 4 * h * h + 3 * h * f
    n = n_mm + 2 * h
    attn_fwd = 2.0 * B * S * S * h
    model_flops = 6.0 * T * (L * n_mm + V * h) + 3.0 * L * attn_fwd
    hw_flops = model_flops + L * (2.0 * n_mm * T + attn_fwd)
    h2d = 2 * (2 * L * n + 2 * V * h)       # bf16 weights: forward + fused recompute/backward (no cache)
    d2h = 4 * (L * n + 2 * V * h)           # fp32 gradients
    return dict(T=T, n=n, n_mm=n_mm, model_flops=model_flops, hw_flops=hw_flops, h2d=h2d, d2h=d2h,
                params=(2 * V * h + L * n))


def smi_gpu_id(local):
    """nvidia-smi id (UUID, else PCI bus id) of this rank's CUDA device, or None."""
    try:
        import torch
        p = torch.cuda.get_device_properties(local)
        u = str(getattr(p, "uuid", "") or "")
        cands = ([u if u.startswith("GPU-") else "GPU-" + u] if u else []) + \
            ["%08X:%02X:%02X.0" % (p.pci_domain_id, p.pci_bus_id, p.pci_device_id)]
    except Exception:
        return None
    for c in cands:
        try:
            r = subprocess.run(["nvidia-smi", "-i", c, "--query-gpu=index", "--format=csv,noheader"],
                               capture_output=True, text=True, timeout=20)
            if r.returncode == 0 and r.stdout.strip():
                return c
        except (OSError, subprocess.TimeoutExpired):
            return None
    return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons of this rank's GPU, sampled during the timed
    region (other GPUs of the node, idle at low clocks, would skew the median)."""

    def __init__(self, gpu_id=None):
        self.rows, self.proc, self.gpu_id = [], None, gpu_id

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi"] + (["-i", self.gpu_id] if self.gpu_id else []) +
                ["--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        sm = [float(r[1]) for r in self.rows if len(r) > 2 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 2 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for i, nme in enumerate(names):
                if len(r) > 5 + i and r[5 + i].lower().startswith("active"):
                    reasons.add(nme)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


class FastClockSampler:
    """SM clock of this rank's GPU every 5 ms through NVML during the timed region. The
    200 ms nvidia-smi samples above mostly land in the GPU's idle gaps of a host-bound
    step (median = the maximum clock); 5 ms samples resolve the GEMM bursts, where the
    power cap pulls the SM clock down to the sustained regime (the clock the kernels'
    roofline peak must match)."""

    def __init__(self, gpu_id, index):
        self.gpu_id, self.index, self.clk, self.stop_, self.t = gpu_id, index, [], False, None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            if self.gpu_id and self.gpu_id.startswith("GPU-"):
                self.h = pynvml.nvmlDeviceGetHandleByUUID(self.gpu_id)
            elif self.gpu_id:
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(self.gpu_id)
            else:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        except Exception:   # NVML absent: the key reports null
            return
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()

    def _loop(self):
        while not self.stop_:
            try:
                self.clk.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            except Exception:
                return
            time.sleep(0.005)

    def stop(self):
        self.stop_ = True
        if self.t is None or not self.clk:
            return None
        self.t.join()
        c = np.array(self.clk, dtype=np.float64)
        return {"sm_mhz_median": float(np.median(c)), "sm_mhz_p10": float(np.percentile(c, 10)),
                "sm_mhz_p90": float(np.percentile(c, 90)), "share_below_1900": float((c < 1900).mean()),
                "samples": int(c.size), "period_ms": 5}


def nvml_index(local):
    """NVML index of the GPU torch calls `local` (CUDA_VISIBLE_DEVICES may remap it)."""
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    ids = [x.strip() for x in vis.split(",") if x.strip()]
    if local < len(ids) and ids[local].isdigit():
        return int(ids[local])
    return local


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), \
        int(os.environ.get("LOCAL_RANK", 0))


def reference_sample(m, steps, warmup):
    """Reference CPU path: block fwd+recompute+bwd and head at full width, T=4."""
    import oracle as O
    ref = O.Reference()
    Bs, Ss = 1, 4
    ctx = ref.bench_create(Bs, Ss, m["hidden"], m["ffn"], m["vocab"])
    try:
        for _ in range(warmup):
            ref.bench_run(ctx)
        per = []
        for _ in range(steps):
            tb, th = ref.bench_run(ctx)
            per.append(m["layers"] * tb + th)
    finally:
        ref.bench_destroy(ctx)
    t_step = float(np.mean(per))            # estimated seconds for T=4 tokens through the model
    tok_s = Bs * Ss / t_step
    sample = (f"reference CPU kernels (oracle/_ref, -O3, 1 thread): one block fwd+recompute+bwd "
              f"and head fwd+CE+bwd at h={m['hidden']} f={m['ffn']} V={m['vocab']} on T={Bs * Ss} "
              f"tokens, x{m['layers']} blocks; estimate, linear in T and L")
    return tok_s, t_step, sample


def host_info():
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


C1_REF = dict(layers=4, hidden=256, ffn=1024, vocab=1024, seq=128, batch=4, n_heads=1)


def measured_c1_reference(steps=3, warmup=1):
    """the reference's full Engine::train_step (proj/src/engine.cpp:426-432),
    bf16-store, measured wall clock at C1 in reference semantics (1 head, no RoPE) on one
    core — the reference step is single-threaded. Measured, not extrapolated."""
    import oracle as O
    m = C1_REF
    c = O.cfg(m["layers"], m["hidden"], m["ffn"], m["vocab"], m["seq"], m["batch"], 1, False, 1, 0.0)
    s = O.Reference().time_train_step(c, True, steps, warmup)
    T = m["batch"] * m["seq"]
    return {"workload": "C1 " + NAMES["c1"].replace("qwen-style", "reference-mode"),
            "shape": m, "steps": steps, "warmup": warmup, "s_per_step": s, "tokens_per_s": T / s,
            "cores": 1, "kind": "reference", **host_info(),
            "def": "oracle/_ref (the reference library, its sources compiled with its Release flags): "
                   "hlm::Engine::train_step in bf16-store mode, wall clock per step"}


def measured_c1_ours(E, steps=3, warmup=2):
    """Our step on the same C1 workload through the public API (host tokens in, loss out,
    host Adam included), wall clock per step — beside the measured reference step."""
    m = C1_REF
    c = E.ModelConfig(m["layers"], m["hidden"], m["ffn"], m["vocab"], m["seq"], m["batch"], k_ckpt=1)
    store = E.Store(c, 1234, "bf16")
    eng = E.Engine(store, E.Arena(c), E.HyperParams(lr=3e-3),
                   E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=4))
    toks = [E.make_copy_task_batch(c, 1235, skip=i) for i in range(warmup + steps)]
    for i in range(warmup):
        eng.train_step(toks[i])
    t0 = time.perf_counter()
    for i in range(steps):
        eng.train_step(toks[warmup + i])
    eng.wait_optimizer()
    s = (time.perf_counter() - t0) / steps
    del eng
    T = m["batch"] * m["seq"]
    return {"s_per_step": s, "tokens_per_s": T / s,
            "def": "Engine.train_step (C ABI) wall clock incl. token H2D, loss D2H and the host Adam"}


def _reference_worker(a):
    m, steps, warmup = a
    sys.path.insert(0, ROOT)
    return reference_sample(m, steps, warmup)


def run_reference(args, m, name):
    """The reference's own CPU implementation (oracle/_ref: its sources compiled with its
    Release flags) on every host core: the reference step is single-threaded, so the
    box's cores run independent replicas of the bounded sample (one block fwd +
    recompute + bwd and the head at full width on 4 tokens, extrapolated to the whole
    model), and their throughputs add up."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    steps = max(1, args.steps)
    warmup = max(0, args.warmup)   # the same W untimed samples as our arm
    cores = int(os.environ.get("HLM_REF_CORES", 0)) or (os.cpu_count() or 1)
    avail = _mem_available()
    if avail:   # ~6.5 GB per replica at C2 width
        per = 4 * (2 * m["vocab"] * m["hidden"] + 4 * m["hidden"] ** 2 + 3 * m["hidden"] * m["ffn"]) * 1.5
        cores = max(1, min(cores, int((avail - 8e9) // per)))
    import multiprocessing as mp
    with mp.get_context("spawn").Pool(cores) as pool:
        res = pool.map(_reference_worker, [(m, steps, warmup)] * cores)
    tok_s = sum(r[0] for r in res)
    t_step = float(np.mean([r[1] for r in res]))
    sample = res[0][2].replace("1 thread", f"{cores} single-threaded replicas, one per core")
    nums = model_numbers(m)
    try:
        mc1 = measured_c1_reference()
    except Exception as ex:
        mc1 = {"error": f"{type(ex).__name__}: {ex}"}
    line = {"metric": METRIC, "value": tok_s, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": steps, "warmup": warmup, "ms_per_step": nums["T"] / tok_s * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp32",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": name, "global_batch": m["batch"], "seq_len": m["seq"],
                       "parallelism": f"cpu-{cores}-replicas"},
            "tflops": nums["model_flops"] / nums["T"] * tok_s / 1e12,
            "cpu_baseline": {"value": tok_s, "unit": "tokens/s", "cores": cores, "kind": "reference",
                             "sample": sample, "per_replica_step_s_for_4_tokens": t_step,
                             "estimate": True, **host_info(), "measured_c1": mc1},
            "e2e": {"value": tok_s, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_hybrid(args, m, nums, E, lib, store, arena, holder, opts, batches, trace, rep):
    """Measured variant, not the headline: the same step with the embedding and the
    first k blocks' FP32 master + Adam state kept in the otherwise idle HBM (device
    Adam, bit-identical to the host Adam; EngineOptions.resident_*). k balances the
    host optimizer time against the GPU's busy time, from the headline run's trace,
    capped by free HBM. The store continues from the headline run's state."""
    import ctypes
    import torch
    L = m["layers"]
    opt = [o for o in trace if o["stream"] == "host" and o["kind"] == "OptStep"]
    dur = lambda o: (o["t_end_us"] - o["t_start_us"]) / 1e6
    blk = [dur(o) for o in opt if 1 <= o["layer"] <= L]
    emb = [dur(o) for o in opt if o["layer"] == 0]
    if not blk:
        return {"error": "no host optimizer ops in the trace"}
    t_blk = float(np.median(blk))
    t_host = sum(dur(o) for o in opt)
    t_gpu = rep["compute_busy_ms"] / 1e3
    # the balance point (host Adam time = GPU busy time, from the headline trace) is a lower
    # bound: a host paced by the GPU idles in the gaps. With the HBM left after the resident
    # state holding saved activations, measured at C2 on one box (k_balance 13-15): slack 2:
    # 15.7 k tok/s, 4: 16.1 k, 6: 16.7 k, 9: 17.2 k (twice), 12: 17.0 k, 14: 16.7 k; so
    # k_balance + 9 (--resident-slack), capped by free HBM
    need = t_host - (emb[0] if emb else 0.0) - t_gpu
    k_balance = int(min(L, max(0, np.ceil(need / t_blk))))
    k = min(L, k_balance + args.resident_slack)
    free, _ = torch.cuda.mem_get_info()
    per_blk, per_emb = 14 * nums["n"], 14 * m["vocab"] * m["hidden"]
    extra = max(0, opts.grad_buffers - 2) * 4 * max(nums["n"], m["vocab"] * m["hidden"])
    room = free - 6e9 - extra
    if room < per_emb:
        return {"error": f"not enough free HBM for the resident embedding ({per_emb / 1e9:.1f} GB needed, "
                         f"{room / 1e9:.1f} GB free after the arena)"}
    k = int(max(0, min(k, (room - per_emb) // per_blk)))
    # HBM left after the resident state keeps the top blocks' forward activations for their
    # backward (no recompute: bit-identical, less GPU time in this GPU-bound variant)
    from paper_2602_04816_b200 import _lib as _L
    dims = _L.HlmBlockDims(m["batch"], m["seq"], m["hidden"], m["ffn"], m["n_heads"], 0)
    act = (int(lib.hlm_cuda_block_acts_bytes(ctypes.byref(dims))) + 255) // 256 * 256
    saved = 0 if args.no_saved_acts else \
        int(max(0, min(L, (room - per_emb - k * per_blk - 2e9) // act)))
    eng = holder.pop()
    eng.sync()
    del eng
    import gc
    gc.collect()
    o2 = E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=opts.n_slab, record_trace=True,
                         grad_buffers=opts.grad_buffers,
                         overlap_optimizer_tail=True, tail_blocks=opts.tail_blocks, resident_embed=True,
                         resident_blocks=k, saved_act_layers=saved,
                         # GPU-bound here: skip the vocab-chunked head's extra head GEMM (it only
                         # serves to start the host Adam of the head earlier)
                         head_piece_vocab=-1)
    eng2 = E.Engine(store, arena, E.HyperParams(lr=1e-4), o2)
    try:
        for i in range(args.warmup):
            eng2.train_step(batches[i])
        lib.hlm_timer_record(2)
        wall0 = time.perf_counter()
        for i in range(args.steps):
            eng2.train_step(batches[args.warmup + i])
        eng2.wait_optimizer()
        lib.hlm_timer_record(3)
        wall = time.perf_counter() - wall0
        dev_s = lib.hlm_timer_elapsed_ms(2, 3) / 1e3
        eng2.sync()
    finally:
        del eng2
    return {"value": nums["T"] * args.steps / dev_s, "unit": "tokens/s", "ms_per_step": dev_s / args.steps * 1e3,
            "e2e": nums["T"] * args.steps / wall, "resident_embed": True, "resident_blocks": k,
            "resident_params": int(m["vocab"] * m["hidden"] + k * nums["n"]),
            "saved_act_layers": saved, "saved_act_bytes": saved * act,
            "balance": {"host_adam_s": t_host, "gpu_busy_s": t_gpu, "host_adam_per_block_s": t_blk,
                        "k_balance": k_balance},
            "def": "not the headline: embedding + blocks 1..k keep FP32 master/m/v in HBM (device Adam, "
                   "bit-identical), the rest host-resident as in the headline; k = k_balance + 9 "
                   "(k_balance: where host Adam time would equal GPU busy time), capped by free HBM; the "
                   "HBM left keeps the top saved_act_layers blocks' forward activations (no recompute)"}


def run_ours(args, m, name):
    rank, world, local = dist_env()
    if args.scaling == "strong":   # global B fixed (8), rows split over the ranks
        if m["batch"] % world:
            raise SystemExit(f"--scaling strong: global batch {m['batch']} not divisible by {world} ranks")
        m = dict(m, batch=m["batch"] // world)
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    # ranks on one host split its cores for their shard of the Adam (init keeps all cores);
    # pinned, the engine sizes each rank's team from its NUMA-local CPU slice itself
    adam_threads = max(1, (os.cpu_count() or 16) // local_world) if world > 1 and args.no_pin else 0
    if args.host_threads > 0:
        adam_threads = args.host_threads
    from paper_2602_04816_b200 import _lib
    from paper_2602_04816_b200 import engine as E

    dp = world > 1 or args.force_dp
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    lib = _lib.blib()
    E.set_device(local)   # before pinning, communicators and the arena
    smi_id = smi_gpu_id(local)
    import ctypes
    lib.hlm_timer_record.argtypes = [ctypes.c_int]
    lib.hlm_timer_elapsed_ms.restype = ctypes.c_double
    lib.hlm_timer_elapsed_ms.argtypes = [ctypes.c_int, ctypes.c_int]
    lib.hlm_cuda_launch_count.restype = ctypes.c_longlong
    lib.hlm_nccl_comm_destroy.argtypes = [ctypes.c_void_p]
    lib.hlm_cuda_bench_block_gemms.argtypes = [ctypes.POINTER(_lib.HlmBlockDims), ctypes.c_int] + \
        [ctypes.POINTER(ctypes.c_double)] * 3
    lib.hlm_ktimer_enable.argtypes = [ctypes.c_int]
    lib.hlm_ktimer_collect.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                       ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]

    # probes on a fresh GPU, before the store / engine exist (after a long host-bound run
    # the same launches read up to 25 % slower): the 12 block GEMMs and the elementwise /
    # norm kernels at the workload's shapes, back to back on random data
    # attention first: measured after the GEMM probe the same launches read 1.4-1.7x slower
    # (the GPU leaves its burst clocks under the GEMMs' power draw for a while)
    attn_probe = attention_probe(lib, m)
    dims = _lib.HlmBlockDims(m["batch"], m["seq"], m["hidden"], m["ffn"], m["n_heads"], 0)
    ew_names = ("rmsnorm_fwd", "rmsnorm_bwd", "swiglu_fwd", "swiglu_bwd", "rope", "cast_bf16")
    ew_gbs, ew_ms = (ctypes.c_double * 6)(), (ctypes.c_double * 6)()
    lib.hlm_cuda_bench_block_ops(ctypes.byref(dims), 20, ew_gbs, ew_ms)
    fl, ms_set, ms_launch = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    lib.hlm_cuda_bench_block_gemms(ctypes.byref(dims), 5, ctypes.byref(fl), ctypes.byref(ms_set),
                                   ctypes.byref(ms_launch))
    gemm_tflops = fl.value / (ms_set.value / 1e3) / 1e12

    cfg = E.ModelConfig(m["layers"], m["hidden"], m["ffn"], m["vocab"], m["seq"], m["batch"],
                        k_ckpt=1, n_heads=m["n_heads"], rope_theta=1e6)
    nums = model_numbers(m)
    t0 = time.time()
    comm_g = comm_w = None
    if dp:
        uids = [E.nccl_unique_id(), E.nccl_unique_id()] if rank == 0 else [None, None]
        if world > 1:
            dist.broadcast_object_list(uids, src=0)
        comm_g = E.nccl_comm(uids[0], world, rank)
        comm_w = E.nccl_comm(uids[1], world, rank)
        shm = f"hlm_bench_{os.environ.get('MASTER_PORT', os.getpid())}"
        import hashlib   # per-run nonce: a stale segment of a crashed run is never attached
        nonce = int.from_bytes(hashlib.blake2b(uids[0], digest_size=8).digest(), "little")
        store = E.Store(cfg, 1234, "bf16", init="parallel", shared=shm, rank=rank, world=world,
                        nonce=nonce)
    else:
        store = E.Store(cfg, 1234, "bf16", init="parallel")
    # HBM weight cache for the backward turnaround: all blocks when they fit next to the arena
    blk = (2 * nums["n"] + 255) // 256 * 256
    cache = min(m["layers"], int(args.cache_gb * 1e9) // blk) * blk
    arena = E.Arena(cfg, device=local, weight_cache_bytes=cache)
    n_slab, tail = pick_slabs(args, m, nums, world, local_world)
    opts = E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=n_slab,
                           grad_buffers=args.grad_buffers, sparse_embed_grad=not args.dense_embed_grad,
                           embed_gather_host=not args.dense_embed_grad, pin_threads=not args.no_pin,
                           record_trace=True, overlap_optimizer_tail=tail >= 0,
                           tail_blocks=max(0, tail), rank=rank, world=world,
                           comm_grad=comm_g, comm_weights=comm_w, host_threads=adam_threads,
                           resident_embed=args.resident_embed, resident_blocks=args.resident_blocks,
                           saved_act_layers=args.saved_act_layers)
    eng = E.Engine(store, arena, E.HyperParams(lr=1e-4), opts)
    setup_s = time.time() - t0
    # one global token stream (reference RNG, global batch = world x local), sliced by rank
    gcfg = E.ModelConfig(m["layers"], m["hidden"], m["ffn"], m["vocab"], m["seq"], m["batch"] * world)
    rows = m["batch"] * m["seq"]
    batches = [E.make_copy_task_batch(gcfg, 1235, skip=i)[rank * rows:(rank + 1) * rows]
               for i in range(args.warmup + args.steps)]

    for i in range(args.warmup):
        eng.train_step(batches[i])
    trace = eng.last_trace()
    if args.dump_trace:
        with open(args.dump_trace, "w") as f:
            for op in trace:
                f.write(json.dumps(op) + "\n")
    if world > 1:
        dist.barrier()
    # per-launch CUDA events around every GEMM / attention launch of the timed steps
    lib.hlm_ktimer_reset()
    lib.hlm_ktimer_enable(1)
    clocks = ClockSampler(smi_id)
    clocks.start()
    fast_clocks = FastClockSampler(smi_id, nvml_index(local))
    fast_clocks.start()
    launches0 = lib.hlm_cuda_launch_count()
    lib.hlm_timer_record(0)
    wall0 = time.perf_counter()
    losses, gpu_ms = [], []
    for i in range(args.steps):
        r = eng.train_step(batches[args.warmup + i])
        losses.append(r.loss)
        gpu_ms.append(r.gpu_ms)
        h2d_step = r.h2d_bytes
        d2h_step = r.d2h_bytes
    eng.wait_optimizer()   # the last step's host optimizer tail is inside the timed region
    lib.hlm_timer_record(1)
    wall = time.perf_counter() - wall0
    launches = (lib.hlm_cuda_launch_count() - launches0) // max(1, args.steps)
    clk = clocks.stop()
    clk["fast"] = fast_clocks.stop()
    if world > 1:   # every rank sampled its own GPU: median of the ranks' medians, union of reasons
        per = [None] * world
        dist.all_gather_object(per, clk)
        meds = [c["sm_mhz"] for c in per if c.get("sm_mhz") is not None]
        clk = {"sm_mhz": float(np.median(meds)) if meds else None,
               "sm_max_mhz": max((c["sm_max_mhz"] for c in per if c.get("sm_max_mhz")), default=None),
               "reasons": sorted(set(r for c in per for r in c["reasons"])),
               "samples": sum(c["samples"] for c in per), "per_rank_sm_mhz": [c.get("sm_mhz") for c in per],
               "fast_per_rank": [c.get("fast") for c in per]}
    lib.hlm_ktimer_enable(0)
    kt = {}
    for kind, kname in ((0, "gemm"), (1, "attn_fwd"), (2, "attn_bwd")):
        ms_k, fl_k, n_k = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        lib.hlm_ktimer_collect(kind, ctypes.byref(ms_k), ctypes.byref(fl_k), ctypes.byref(n_k))
        kt[kname] = {"ms": ms_k.value, "flops": fl_k.value, "launches": n_k.value,
                     "tflops": fl_k.value / (ms_k.value / 1e3) / 1e12 if ms_k.value > 0 else None}
    ew_step = {}
    for kind, kname in ((3, "rmsnorm_fwd"), (4, "rmsnorm_bwd"), (5, "swiglu_fwd"), (6, "swiglu_bwd"),
                        (7, "rope"), (8, "cast_bf16")):
        ms_k, by_k, n_k = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        lib.hlm_ktimer_collect(kind, ctypes.byref(ms_k), ctypes.byref(by_k), ctypes.byref(n_k))
        ew_step[kname] = {"ms": ms_k.value, "bytes": by_k.value, "launches": n_k.value,
                          "gbs": by_k.value / (ms_k.value / 1e3) / 1e9 if ms_k.value > 0 else None}
    lib.hlm_ktimer_reset()
    dev_s = lib.hlm_timer_elapsed_ms(0, 1) / 1e3
    if world > 1:
        import torch
        t = torch.tensor([dev_s])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s = float(t.item())
    step_s = dev_s / args.steps
    value = world * nums["T"] * args.steps / dev_s
    e2e = world * nums["T"] * args.steps / wall

    # per-step overlap / bandwidth / protocol check from the measured trace (last warm-up step)
    from paper_2602_04816_b200.trace import overlap_report, validate_trace
    rep = overlap_report(trace)
    h2d_gbs, d2h_gbs, overlap = rep["h2d_gbs"], rep["d2h_gbs"], rep["overlap"]
    violations = validate_trace(trace, m["layers"])
    host_ops = [o for o in trace if o["stream"] == "host" and o["kind"] == "OptStep"]
    adam_s = sum(o["t_end_us"] - o["t_start_us"] for o in host_ops) / 1e6
    gpu_span_s = float(np.mean(gpu_ms)) / 1e3   # step-start .. step-end events on the compute stream

    hbm, tf_burst, tf_sus, peak_kind = peaks()
    # DRAM bytes per launch of one block's 12 GEMMs (fused epilogues, as timed in-step) from
    # the committed ncu --set full capture of the same kernels
    tp = os.path.join(ROOT, "profiles", "r02", "r02_gemm_block_traffic.json")
    gemm_traffic = json.load(open(tp)) if os.path.exists(tp) and m["hidden"] == 3584 else {}
    elementwise = {k: {"gbs": ew_gbs[i], "ms": ew_ms[i], "frac": ew_gbs[i] / hbm}
                   for i, k in enumerate(ew_names)}
    for k, v in ew_step.items():
        v["frac"] = (v["gbs"] or 0) / hbm

    t_roof = max(nums["hw_flops"] / (tf_sus * 1e12), nums["h2d"] / (PCIE_ASSUMED_GBS * 1e9),
                 nums["d2h"] / (PCIE_ASSUMED_GBS * 1e9))
    # stricter per-phase roofline: forward max(flops, weight H2D) + backward
    # max(recompute + backward flops, gradient D2H); with the HBM weight cache the backward
    # streams no weights
    attn_fwd = 2.0 * m["batch"] * m["seq"] ** 2 * m["hidden"]
    fl_fwd = m["layers"] * (2.0 * nums["n_mm"] * nums["T"] + attn_fwd) + 2.0 * nums["T"] * m["vocab"] * m["hidden"]
    fl_bwd = nums["hw_flops"] - fl_fwd
    t_fwd = max(fl_fwd / (tf_sus * 1e12), h2d_step / (PCIE_ASSUMED_GBS * 1e9))
    t_bwd = max(fl_bwd / (tf_sus * 1e12), nums["d2h"] / (PCIE_ASSUMED_GBS * 1e9))
    # host DRAM roofline: every parameter moves 30 B through the host Adam (g, w, m, v in;
    # w, m, v, bf16 shadow out) + 4 B of gradient DMA written + 2 B per weight DMA pass read
    lib.hlm_host_triad_gbs.restype = ctypes.c_double
    lib.hlm_host_triad_gbs.argtypes = [ctypes.c_int64, ctypes.c_int]
    host_bw = lib.hlm_host_triad_gbs(1 << 30, 5) if rank == 0 else None
    # 26 B/param of Adam state traffic (w, m, v read + written, bf16 shadow written) + the
    # gradient bytes twice (DMA write, Adam read) + the weight DMA read
    host_bytes = nums["params"] * 26 + 2 * d2h_step + h2d_step
    # STREAM counts 3 arrays for a triad but the DRAM also serves the write-allocate read of
    # `a`: raw bandwidth = 4/3 x triad. Our traffic is raw (non-temporal shadow stores, DMA
    # writes whole lines, w/m/v are read before written).
    raw_bw = host_bw * 4.0 / 3.0 if host_bw else None
    t_host = host_bytes / (raw_bw * 1e9) if raw_bw else None

    cpu_baseline = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            tok_s, _, sample = reference_sample(m, 1, 0)
            cpu_baseline = {"value": tok_s, "unit": "tokens/s", "cores": 1, "kind": "reference",
                            "sample": sample}
        except Exception as ex:   # reference lib absent -> say so
            cpu_baseline = {"value": None, "unit": "tokens/s", "cores": 1, "kind": "reference",
                            "sample": f"unavailable: {ex}"}

    hybrid = None
    if world == 1 and not args.no_hybrid and not dp:
        try:
            holder = [eng]
            eng = None   # the headline engine (and its pinned slabs) must be gone before the variant's
            hybrid = run_hybrid(args, m, nums, E, lib, store, arena, holder, opts, batches, trace, rep)
        except Exception as ex:
            hybrid = {"error": f"{type(ex).__name__}: {ex}"}

    if cpu_baseline is not None:
        cpu_baseline.update(estimate=True, **host_info())
        try:   # the reference's full train_step measured at C1 beside ours
            ref_c1 = measured_c1_reference()
            ours_c1 = measured_c1_ours(E)
            ref_c1["ours"] = ours_c1
            ref_c1["speedup_e2e"] = ref_c1["s_per_step"] / ours_c1["s_per_step"]
            cpu_baseline["measured_c1"] = ref_c1
        except Exception as ex:
            cpu_baseline["measured_c1"] = {"error": f"{type(ex).__name__}: {ex}"}

    if hybrid and "ms_per_step" in hybrid:
        hs = hybrid["ms_per_step"] / 1e3
        hybrid["step_roofline_frac"] = t_roof / hs
        hybrid["phase_roofline_frac"] = (t_fwd + t_bwd) / hs
    if rank != 0:
        if world > 1:
            dist.barrier()
        del eng
        for c in (comm_g, comm_w):
            if c is not None:
                lib.hlm_nccl_comm_destroy(c)
        return
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": step_s * 1e3, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic copy-task tokens, random-init weights (parallel trunc-normal 0.02)",
        "config": {"workload": name, "global_batch": m["batch"] * world, "seq_len": m["seq"],
                   "tokens_per_step": nums["T"] * world, "params": nums["params"],
                   "parallelism": f"dp{world}" if (world > 1 or dp) else "single-gpu",
                   "n_heads": m["n_heads"], "k_ckpt": 1, "l2": "inputs larger than L2 (weights "
                   "streamed from host every step)",
                   "gradient_slabs": n_slab, "optimizer_tail_blocks": tail,
                   "hbm_resident_optimizer": {"embed": bool(args.resident_embed),
                                              "blocks": args.resident_blocks}},
        "tflops": nums["model_flops"] / step_s / 1e12,
        "hw_tflops": nums["hw_flops"] / step_s / 1e12,
        "e2e": {"value": e2e, "unit": "tokens/s",
                "h2d_bytes_per_step": int(h2d_step + 8 * nums["T"]),
                "d2h_bytes_per_step": int(d2h_step + 4 * nums["T"]),
                "def": "wall clock around the same K Engine.train_step calls (C ABI hlm_engine_train_step) "
                       "plus the final optimizer drain: every step copies its tokens / targets H2D from "
                       "pinned host memory, streams the BF16 weights H2D from the host store, copies the "
                       "FP32 gradients and the per-row losses D2H and runs the host Adam. In this design "
                       "the inputs (weights) live on the host, so `value` (CUDA events around the same "
                       "region) and e2e measure the same host-bound work and differ only by clock"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "tensor", "kernel": "gemm_sm100 (tcgen05/TMA): every GEMM launch of the timed "
                                                  "steps (block fwd / recompute / dgrad / wgrad, head)",
                     "achieved": kt["gemm"]["tflops"], "peak": tf_sus, "unit": "TFLOP/s",
                     "frac": (kt["gemm"]["tflops"] or 0) / tf_sus,
                     "peak_kind": f"{peak_kind} sustained: the GEMMs are timed inside a long step whose "
                                  "GEMM bursts run at power-capped clocks (clocks.fast: 5 ms NVML samples "
                                  "of the timed region; tools/instep_probe.py: the same in-step GEMM time "
                                  "with the host Adam off, so host contention is not the cause)",
                     "frac_of_burst": (kt["gemm"]["tflops"] or 0) / tf_burst, "peak_burst": tf_burst,
                     "def": "algorithmic GEMM flops (2MNK per launch) / CUDA-event time of the launches, "
                            "on the compute stream, over the timed steps",
                     "launches_per_step": kt["gemm"]["launches"] / max(1, args.steps),
                     "ms_per_launch": kt["gemm"]["ms"] / max(1, kt["gemm"]["launches"]),
                     "share_of_step": kt["gemm"]["ms"] / 1e3 / max(1e-9, dev_s),
                     "traffic": gemm_traffic.get("dram_bytes_per_launch"),
                     "algorithmic_bytes_per_launch": gemm_traffic.get("algorithmic_bytes_per_launch"),
                     "traffic_source": gemm_traffic.get("source"),
                     "probe": {"achieved": gemm_tflops, "frac_of_burst": gemm_tflops / tf_burst,
                               "ms_per_launch": ms_launch.value,
                               "def": "the 12 block GEMMs at the workload shapes on random data, "
                                      "back to back (hlm_cuda_bench_block_gemms)"}},
        "attention_roofline": {k: dict(kt[k], frac=(kt[k]["tflops"] or 0) / tf_sus, peak=tf_sus,
                                       frac_of_burst=(kt[k]["tflops"] or 0) / tf_burst, peak_burst=tf_burst,
                                       standalone=attn_probe.get(k),
                                       note="in-step: CUDA events around each attention call of the timed steps; "
                                            "each call follows a GEMM burst and runs at the clock the power "
                                            "cap left (clocks.fast); standalone: the same call back to back at "
                                            "the workload shape, clocks near maximum (fractions of burst); the "
                                            "ncu launch list (profiles/r02/r02_launches_c2.csv) has the kernels "
                                            "within 7 % of standalone")
                               for k in ("attn_fwd", "attn_bwd")},
        "elementwise_roofline": {"peak_gbs": hbm, "unit": "GB/s", "in_step": ew_step, "probe": elementwise,
                                 "note": "in_step launches run between GEMM bursts at the power-capped SM "
                                         "clock (clocks.fast) and each event pair adds its launch latency to "
                                         "a 25-300 us kernel; per-kernel durations from ncu (profiles/r02/"
                                         "r02_launches_c2.csv) give 0.95-1.03 of HBM for these kernels",
                                 "def": "algorithmic bytes (each tensor read/written once) / CUDA-event time; "
                                        "in_step: every launch of the timed steps; probe: back-to-back "
                                        "launches at the workload shape after the steps"},
        "step_roofline": {"t_roof_s": t_roof, "t_step_s": step_s, "frac": t_roof / step_s,
                          "def": "max(HW_FLOPS/sustained bf16, H2D/55GB/s, D2H/55GB/s)"},
        "phase_roofline": {"t_fwd_s": t_fwd, "t_bwd_s": t_bwd, "t_roof_s": t_fwd + t_bwd,
                           "frac": (t_fwd + t_bwd) / step_s,
                           "def": "max(fwd flops/sustained bf16, measured weight H2D bytes/55GB/s) + "
                                  "max(recompute+bwd flops/sustained bf16, D2H bytes/55GB/s)"},
        "host_roofline": {"host_bytes_per_step": int(host_bytes), "triad_gbs": host_bw,
                          "raw_dram_gbs": raw_bw, "t_host_s": t_host,
                          "frac": (t_host / step_s) if t_host else None,
                          "def": "(26 B/param host Adam state + gradient bytes x 2 (DMA write, Adam read) + "
                                 "weight DMA bytes) / (4/3 x measured 16-thread STREAM triad = raw DRAM "
                                 "bandwidth)"},
        "stream": {"h2d_gbs": h2d_gbs, "d2h_gbs": d2h_gbs, "overlap": overlap,
                   "h2d_overlap": rep["h2d_overlap"], "h2d_exposed_s": rep["h2d_exposed_ms"] / 1e3,
                   "d2h_overlap": rep["d2h_overlap"], "d2h_exposed_s": rep["d2h_exposed_ms"] / 1e3,
                   "transfer_overlap": rep["transfer_overlap"],
                   "compute_idle_s": rep["compute_idle_ms"] / 1e3,
                   "overlap_def": "overlap: share of H2D + D2H busy time with the compute stream busy; "
                                  "h2d_overlap: 1 - (compute idle while a weight transfer it waits on "
                                  "is in flight) / H2D busy time; d2h_overlap: the same for a backward "
                                  "waiting on its gradient buffer's D2H; transfer_overlap: both "
                                  "directions, 1 - exposed transfer / transfer (SURVEY 8d)",
                   "gpu_span_s": gpu_span_s, "compute_busy_s": rep["compute_busy_ms"] / 1e3,
                   "host_adam_s": adam_s,
                   "h2d_bytes_measured": int(h2d_step), "trace_violations": len(violations)},
        "clocks": clk, "cpu_baseline": cpu_baseline, "hbm_resident_variant": hybrid,
        "loss": [float(x) for x in losses], "setup_s": setup_s,
    }
    if world > 1:
        dist.barrier()
    del eng
    for c in (comm_g, comm_w):
        if c is not None:
            lib.hlm_nccl_comm_destroy(c)
    return line


WIDE_POINTS = {"c3": (4, 8), "c4": (2, 4, 6), "c5": (1, 2)}
WIDE_DEFAULT = ("c4", "c5")   # the north-star target width and the largest; c3 on request (--wide-only)


def run_wide(args):
    """N1: the 72B-width (C4) and 120B-width (C5) decoders do not fit a 196 GB
    host at full depth (1.15 / 1.69 TB of FP32 master + Adam), so each is measured at full
    width over a depth sweep — same step, same options as the headline, each point in its
    own process after the headline's store is gone — and the full-depth step is projected
    from a per-layer fit t(L) = a + b L. Projections are labelled as such."""
    out = {}
    for cfg, depths in WIDE_POINTS.items():
        if cfg not in (args.wide_only.split(",") if args.wide_only else WIDE_DEFAULT):
            continue
        pts = []
        for L in depths:
            cmd = [sys.executable, os.path.abspath(__file__), "--config", cfg, "--layers", str(L),
                   "--steps", str(args.wide_steps), "--warmup", "2", "--no-hybrid",
                   "--no-cpu-baseline", "--no-wide"]
            t0 = time.time()
            r = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
            lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
            if r.returncode != 0 or not lines:
                pts.append({"layers": L, "error": (r.stderr or r.stdout)[-400:]})
                continue
            d = json.loads(lines[-1])
            pts.append({"layers": L, "params": d["config"]["params"], "value": d["value"],
                        "ms_per_step": d["ms_per_step"], "tflops": d["tflops"],
                        "e2e": d["e2e"]["value"], "h2d_overlap": d["stream"]["h2d_overlap"],
                        "transfer_overlap": d["stream"].get("transfer_overlap"),
                        "overlap": d["stream"]["overlap"], "host_adam_s": d["stream"]["host_adam_s"],
                        "compute_busy_s": d["stream"]["compute_busy_s"],
                        "gemm_tflops_in_step": d["roofline"]["achieved"],
                        "gemm_frac": d["roofline"]["frac"],
                        "attn_fwd_tflops": d["attention_roofline"]["attn_fwd"]["tflops"],
                        "attn_bwd_tflops": d["attention_roofline"]["attn_bwd"]["tflops"],
                        "step_roofline_frac": d["step_roofline"]["frac"],
                        "host_roofline_frac": d["host_roofline"]["frac"],
                        "clocks": d["clocks"], "wall_s": time.time() - t0})
        ok = [p for p in pts if "ms_per_step" in p]
        entry = {"points": pts, "width": {k: CONFIGS[cfg][k] for k in
                                          ("hidden", "ffn", "vocab", "seq", "batch", "n_heads")}}
        if len(ok) >= 2:
            Ls = np.array([p["layers"] for p in ok], float)
            ts = np.array([p["ms_per_step"] / 1e3 for p in ok])
            b, a = np.polyfit(Ls, ts, 1)
            full = dict(CONFIGS[cfg])
            nums = model_numbers(full)
            t_full = a + b * full["layers"]
            _, _, tf_sus, _ = peaks()
            t_roof = max(nums["hw_flops"] / (tf_sus * 1e12), nums["h2d"] / (PCIE_ASSUMED_GBS * 1e9),
                         nums["d2h"] / (PCIE_ASSUMED_GBS * 1e9))
            entry["projection"] = {
                "label": "PROJECTION from the measured depth sweep (not a measured step)",
                "fit": {"a_s": a, "b_s_per_layer": b,
                        "max_residual_s": float(np.max(np.abs(a + b * Ls - ts)))},
                "layers": full["layers"], "params": nums["params"], "t_step_s": t_full,
                "tokens_per_s": nums["T"] / t_full, "tflops": nums["model_flops"] / t_full / 1e12,
                "north_star_roofline": {"t_roof_s": t_roof, "frac": t_roof / t_full,
                                        "def": "max(HW_FLOPS/sustained bf16, H2D/55GB/s, D2H/55GB/s)"},
                "host_store_bytes": nums["params"] * 14}
        out[cfg] = entry
    return out


def attention_probe(lib, m, iters=10):
    """The attention kernels alone at the workload shape (random q/k/v/dO, CUDA events,
    back to back, before the store exists): the standalone reference point for the in-step
    attention numbers, which run at the clocks the GEMMs leave."""
    import ctypes
    import torch
    from paper_2602_04816_b200 import _lib
    B, S, H, h = m["batch"], m["seq"], m["n_heads"], m["hidden"]
    T = B * S
    try:
        q, k, v, do = (torch.randn(T, h, device="cuda").bfloat16() for _ in range(4))
        o, dq, dk, dv = (torch.empty_like(q) for _ in range(4))
        lse, ds = torch.empty(B * H * S, device="cuda"), torch.empty(B * H * S, device="cuda")
        d = _lib.HlmBlockDims(B, S, h, m["ffn"], H, 0)
        vp = lambda t: ctypes.c_void_p(t.data_ptr())
        fwd = lambda: _lib.check(lib.hlm_cuda_attention_fwd(ctypes.byref(d), vp(q), vp(k), vp(v), vp(o), vp(lse), h,
                                                             None))
        bwd = lambda: _lib.check(lib.hlm_cuda_attention_bwd(ctypes.byref(d), vp(q), vp(k), vp(v), vp(o), vp(do),
                                                             vp(lse), vp(ds), vp(dq), vp(dk), vp(dv), h, None))
        out = {}
        fl = 2.0 * B * S * S * h   # causal: the reference's flop count
        for name, fn, work in (("attn_fwd", fwd, fl), ("attn_bwd", bwd, 2.5 * fl)):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(iters):
                fn()
            b.record()
            torch.cuda.synchronize()
            ms = a.elapsed_time(b) / iters
            out[name] = {"ms": ms, "tflops": work / (ms / 1e3) / 1e12}
        del q, k, v, do, o, dq, dk, dv, lse, ds
        torch.cuda.empty_cache()
        return out
    except Exception as ex:   # a probe, not the measurement: never fail the bench on it
        return {"error": f"{type(ex).__name__}: {ex}"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--slabs", type=int, default=0,
                    help="pinned gradient slabs (0: auto = layers + 4, capped by free host memory)")
    ap.add_argument("--tail-blocks", type=int, default=-2,
                    help="blocks optimised after the embedding, overlapping the next forward "
                         "(-1: off, -2: auto = every block the slab pool can hold)")
    ap.add_argument("--cache-gb", type=float, default=60.0,
                    help="HBM weight cache (block tiles resident between forward and backward)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--grad-buffers", type=int, default=8,
                    help="device fp32 gradient buffers (2 = the arena's; more let the backward run "
                         "ahead of a slow D2H)")
    ap.add_argument("--dense-embed-grad", action="store_true",
                    help="stream the whole (V, h) embedding table / gradient (default: only the batch's "
                         "token rows: zero-copy gather in the forward, row-sparse gradient)")
    ap.add_argument("--host-threads", type=int, default=0,
                    help="OpenMP threads of the host optimizer (0: all cores / cores per local rank)")
    ap.add_argument("--no-pin", action="store_true", help="leave the host optimizer threads unpinned")
    ap.add_argument("--no-hybrid", action="store_true",
                    help="skip the measured HBM-resident-optimizer variant reported beside the headline")
    ap.add_argument("--resident-slack", type=int, default=9,
                    help="variant: resident blocks beyond the host/GPU balance point")
    ap.add_argument("--no-saved-acts", action="store_true",
                    help="variant: recompute every block instead of keeping spare-HBM activations")
    ap.add_argument("--saved-act-layers", type=int, default=0,
                    help="top blocks whose forward activations stay in HBM (no recompute)")
    ap.add_argument("--resident-blocks", type=int, default=0,
                    help="blocks 1..N keep FP32 master + Adam state in HBM (device Adam, no streaming)")
    ap.add_argument("--resident-embed", action="store_true",
                    help="the embedding table keeps FP32 master + Adam state in HBM")
    ap.add_argument("--force-dp", action="store_true",
                    help="use the data-parallel code path (NCCL, shared store) even at world 1")
    ap.add_argument("--dump-trace", default="", help="write the last warm-up step's measured trace (JSONL)")
    ap.add_argument("--layers", type=int, default=0,
                    help="partial depth of the config's full-width decoder (C3-C5 do not fit a 196 GB "
                         "host at full depth); the workload name says so")
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="weak: B rows per GPU (global batch grows with N); strong: the config's global "
                         "batch split over the N ranks (SURVEY 8d)")
    ap.add_argument("--no-wide", action="store_true",
                    help="skip the C4 / C5 full-width depth sweeps reported beside a C2 headline")
    ap.add_argument("--wide-only", default="", help="comma list of wide configs to sweep (default c4,c5; c3 too)")
    ap.add_argument("--wide-steps", type=int, default=3, help="timed steps per wide point")
    args = ap.parse_args()
    m = dict(CONFIGS[args.config])
    name = NAMES[args.config]
    if args.layers > 0 and args.layers != m["layers"]:
        name = f"{name}-first{args.layers}of{m['layers']}layers"
        m["layers"] = args.layers
    if args.impl == "reference":
        run_reference(args, m, name)
        return
    line = run_ours(args, m, name)
    if line is None:
        return
    if (not args.no_wide and args.config == "c2" and args.layers == 0 and line["n_gpus"] == 1
            and not args.force_dp):
        import gc
        gc.collect()
        try:
            line["wide"] = run_wide(args)
        except Exception as ex:
            line["wide"] = {"error": f"{type(ex).__name__}: {ex}"}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
