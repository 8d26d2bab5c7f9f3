"""Python mirror of the host engine (ctypes over include/hlm_cuda.h).

Same surface as the reference's C++ API and Python module
(proj/include/hlm/engine.hpp, host_store.hpp, device_arena.hpp, trainer.hpp;
proj/python/hlm/__init__.py): ``ModelConfig``, ``HyperParams``,
``EngineOptions``, ``Store`` (build_store), ``Arena`` (DeviceArena),
``Engine`` (train_step + phase API), ``make_copy_task_batch`` and ``train``.
Errors surface as the reference's exception types (ConfigError ->
ValueError, ArenaOom -> MemoryError, out_of_range -> IndexError ...).
"""

import ctypes
import json

import numpy as np

from . import _lib

_vp = ctypes.c_void_p
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")


class HlmConfigError(ValueError):
    pass


class ArenaOom(MemoryError):
    pass


class ProtocolError(RuntimeError):
    pass


class NumericsError(ArithmeticError):
    pass


class CudaError(RuntimeError):
    pass


_ERRORS = {2: HlmConfigError, 3: ArenaOom, 4: ProtocolError, 5: NumericsError, 6: IndexError,
           7: CudaError, 8: RuntimeError}


def _check(rc):
    if rc != 0:
        msg = _lib.lib().hlm_cuda_last_error().decode()
        raise _ERRORS.get(rc, RuntimeError)(msg)


class ModelConfig(ctypes.Structure):
    _fields_ = [("layers", ctypes.c_int64), ("hidden", ctypes.c_int64), ("ffn", ctypes.c_int64),
                ("vocab", ctypes.c_int64), ("seq", ctypes.c_int64), ("batch", ctypes.c_int64),
                ("k_ckpt", ctypes.c_int64), ("tie_embeddings", ctypes.c_int32),
                ("n_heads", ctypes.c_int32), ("rope_theta", ctypes.c_double)]

    def __init__(self, layers, hidden, ffn, vocab, seq, batch, k_ckpt=1, tie_embeddings=False,
                 n_heads=1, rope_theta=0.0):
        super().__init__(layers, hidden, ffn, vocab, seq, batch, k_ckpt, int(tie_embeddings),
                         n_heads, rope_theta)

    @property
    def rows(self):
        return self.batch * self.seq

    def block_params(self):
        h, f = self.hidden, self.ffn
        return 4 * h * h + 3 * h * f + 2 * h

    def total_params(self):
        t = self.vocab * self.hidden * (1 if self.tie_embeddings else 2)
        return t + self.layers * self.block_params()


class HyperParams(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("weight_decay", ctypes.c_double)]

    def __init__(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0):
        super().__init__(lr, beta1, beta2, eps, weight_decay)


class EngineOptions(ctypes.Structure):
    _fields_ = [("eager_optim", ctypes.c_int32), ("threaded_accum", ctypes.c_int32),
                ("n_slab", ctypes.c_int64), ("accum_delay_us", ctypes.c_int64),
                ("skip_optimizer", ctypes.c_int32), ("fused_recompute", ctypes.c_int32),
                ("record_trace", ctypes.c_int32), ("block_flags", ctypes.c_int32),
                ("overlap_optimizer_tail", ctypes.c_int32), ("tail_blocks", ctypes.c_int32),
                ("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("comm_grad", ctypes.c_void_p),
                ("comm_weights", ctypes.c_void_p), ("host_threads", ctypes.c_int32),
                ("resident_embed", ctypes.c_int32), ("resident_blocks", ctypes.c_int64),
                ("head_piece_vocab", ctypes.c_int64), ("piece_elems", ctypes.c_int64),
                ("grad_buffers", ctypes.c_int64), ("sparse_embed_grad", ctypes.c_int32),
                ("embed_gather_host", ctypes.c_int32), ("no_pin_threads", ctypes.c_int32),
                ("reserved_transit_blocks", ctypes.c_int64), ("saved_act_layers", ctypes.c_int64)]

    def __init__(self, eager_optim=False, threaded_accum=False, n_slab=12, accum_delay_us=0,
                 skip_optimizer=False, fused_recompute=True, record_trace=True, block_flags=0,
                 overlap_optimizer_tail=False, tail_blocks=2, rank=0, world=1, comm_grad=None,
                 comm_weights=None, host_threads=0, resident_embed=False, resident_blocks=0,
                 head_piece_vocab=0, piece_elems=0, grad_buffers=2, sparse_embed_grad=False,
                 embed_gather_host=False, pin_threads=True, saved_act_layers=0):
        super().__init__(int(eager_optim), int(threaded_accum), n_slab, accum_delay_us,
                         int(skip_optimizer), int(fused_recompute), int(record_trace), block_flags,
                         int(overlap_optimizer_tail), tail_blocks, rank, world,
                         comm_grad.value if isinstance(comm_grad, ctypes.c_void_p) else comm_grad,
                         comm_weights.value if isinstance(comm_weights, ctypes.c_void_p)
                         else comm_weights, host_threads, int(resident_embed), resident_blocks,
                         head_piece_vocab, piece_elems, grad_buffers, int(sparse_embed_grad),
                         int(embed_gather_host), int(not pin_threads), 0, saved_act_layers)


class StepResult(ctypes.Structure):
    _fields_ = [("loss", ctypes.c_double), ("h2d_bytes", ctypes.c_int64),
                ("d2h_bytes", ctypes.c_int64), ("recompute_forwards", ctypes.c_int64),
                ("gpu_ms", ctypes.c_double), ("arena_committed", ctypes.c_int64),
                ("arena_peak", ctypes.c_int64), ("host_total", ctypes.c_int64),
                ("slab_max_in_use", ctypes.c_int64)]


FIELD_MASTER, FIELD_M, FIELD_V, FIELD_GRADS, FIELD_SHADOW = range(5)
_ready = False


def _L():
    global _ready
    L = _lib.lib()
    if not _ready:
        P = ctypes.POINTER
        L.hlm_store_create.argtypes = [P(ModelConfig), ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, P(_vp)]
        L.hlm_store_destroy.argtypes = [_vp]
        L.hlm_store_total_params.argtypes = [_vp]
        L.hlm_store_total_params.restype = ctypes.c_int64
        L.hlm_store_adam_steps.argtypes = [_vp]
        L.hlm_store_adam_steps.restype = ctypes.c_int64
        L.hlm_store_export.argtypes = [_vp, ctypes.c_int, _f32p]
        L.hlm_store_import_master.argtypes = [_vp, _f32p]
        L.hlm_store_bitwise_equal.argtypes = [_vp, _vp]
        L.hlm_store_adam_step.argtypes = [_vp, _f32p, P(HyperParams), ctypes.c_int64]
        L.hlm_store_adam_embed_rows.argtypes = [_vp, np.ctypeslib.ndpointer(np.int32), ctypes.c_int64, _f32p,
                                                P(HyperParams), ctypes.c_int64]
        L.hlm_store_create_shared.argtypes = [P(ModelConfig), ctypes.c_uint64, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                                              ctypes.c_int, ctypes.c_int, ctypes.c_uint64, P(_vp)]
        L.hlm_store_adam_shard.argtypes = [_vp, _f32p, P(HyperParams), ctypes.c_int64, ctypes.c_int,
                                           ctypes.c_int]
        L.hlm_store_tile_version.argtypes = [_vp, ctypes.c_int64]
        L.hlm_store_tile_version.restype = ctypes.c_int64
        L.hlm_store_save.argtypes = [_vp, ctypes.c_char_p]
        L.hlm_store_load.argtypes = [_vp, ctypes.c_char_p]
        L.hlm_store_save_hlm1.argtypes = [_vp, ctypes.c_char_p]
        L.hlm_run_training_store.argtypes = [_vp, P(HyperParams), ctypes.c_uint64, ctypes.c_int64,
                                             P(EngineOptions), _f64p]
        L.hlm_nccl_unique_id.argtypes = [ctypes.c_char_p]
        L.hlm_nccl_comm_create.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, P(_vp)]
        L.hlm_nccl_comm_destroy.argtypes = [_vp]
        L.hlm_arena_create.argtypes = [P(ModelConfig), ctypes.c_int64, ctypes.c_int, P(_vp)]
        L.hlm_arena_create_ex.argtypes = [P(ModelConfig), ctypes.c_int64, ctypes.c_int,
                                          ctypes.c_int64, P(_vp)]
        L.hlm_arena_destroy.argtypes = [_vp]
        L.hlm_arena_footprint.argtypes = [P(ModelConfig), np.ctypeslib.ndpointer(np.int64)]
        L.hlm_engine_create.argtypes = [_vp, _vp, P(HyperParams), P(EngineOptions), P(_vp)]
        L.hlm_engine_destroy.argtypes = [_vp]
        L.hlm_engine_train_step.argtypes = [_vp, _i32p, _i32p, P(StepResult)]
        L.hlm_engine_sync.argtypes = [_vp]
        L.hlm_engine_wait_optimizer.argtypes = [_vp]
        L.hlm_engine_begin_step.argtypes = [_vp, _i32p, _i32p]
        L.hlm_engine_forward.argtypes = [_vp]
        L.hlm_engine_anchor_loss.argtypes = [_vp, P(ctypes.c_double)]
        L.hlm_engine_backward.argtypes = [_vp]
        L.hlm_engine_finish_step.argtypes = [_vp, P(StepResult)]
        L.hlm_engine_debug_hidden.argtypes = [_vp, _f32p]
        L.hlm_engine_last_trace.argtypes = [_vp, ctypes.c_char_p, ctypes.c_size_t,
                                            P(ctypes.c_size_t)]
        L.hlm_make_copy_task_batch.argtypes = [P(ModelConfig), ctypes.c_uint64, ctypes.c_int64,
                                               _i32p]
        L.hlm_run_training.argtypes = [P(ModelConfig), P(HyperParams), ctypes.c_uint64,
                                       ctypes.c_int, ctypes.c_int64, P(EngineOptions), _f64p,
                                       P(StepResult)]
        _ready = True
    return L


class Store:
    """Host parameter store (build_store). dtype 'bf16' | 'fp32' (initial rounding);
    init 'reference' (bit-identical to the reference) | 'parallel'."""

    def __init__(self, cfg, seed, dtype="bf16", init="reference", pin=True, shared=None, rank=0,
                 world=1, nonce=0):
        """shared: name of a /dev/shm object for a one-process-per-GPU store
        (rank 0 creates and initialises it, other ranks attach); nonce: per-run token
        shared by all ranks (a stale segment of another run is never attached)."""
        self.cfg = cfg
        h = _vp()
        dt, im = (1 if dtype == "fp32" else 0), (1 if init == "parallel" else 0)
        if shared:
            _check(_L().hlm_store_create_shared(ctypes.byref(cfg), seed, dt, im, int(pin),
                                                shared.encode(), rank, world, nonce, ctypes.byref(h)))
        else:
            _check(_L().hlm_store_create(ctypes.byref(cfg), seed, dt, im, int(pin), ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            _L().hlm_store_destroy(self.h)
            self.h = None

    @property
    def total_params(self):
        return _L().hlm_store_total_params(self.h)

    @property
    def adam_steps(self):
        return _L().hlm_store_adam_steps(self.h)

    def export(self, field=FIELD_MASTER):
        out = np.empty(self.total_params, np.float32)
        _check(_L().hlm_store_export(self.h, field, out))
        return out

    def weights(self):
        return self.export(FIELD_MASTER)

    def grads(self):
        return self.export(FIELD_GRADS)

    def import_master(self, w):
        _check(_L().hlm_store_import_master(self.h, np.ascontiguousarray(w, np.float32)))

    def adam_step(self, grads, hyper, t):
        _check(_L().hlm_store_adam_step(self.h, np.ascontiguousarray(grads, np.float32),
                                        ctypes.byref(hyper), t))

    def adam_embed_rows(self, rows, compact, hyper, t):
        rows = np.ascontiguousarray(rows, np.int32)
        _check(_L().hlm_store_adam_embed_rows(self.h, rows, len(rows),
                                              np.ascontiguousarray(compact, np.float32).ravel(),
                                              ctypes.byref(hyper), t))

    def bitwise_equal(self, other):
        return bool(_L().hlm_store_bitwise_equal(self.h, other.h))

    def save(self, path):
        _check(_L().hlm_store_save(self.h, str(path).encode()))

    def load(self, path):
        """HLM2, or a reference HLM1 file (master := its weights, m / v / step restored)."""
        _check(_L().hlm_store_load(self.h, str(path).encode()))

    def save_hlm1(self, path):
        """The reference's HLM1 container (its load_checkpoint reads it)."""
        _check(_L().hlm_store_save_hlm1(self.h, str(path).encode()))

    def run_training(self, hyper, seed, steps, options=None):
        """run_training on this store (resume-aware: replays the data stream)."""
        losses = np.empty(steps, np.float64)
        _check(_L().hlm_run_training_store(self.h, ctypes.byref(hyper), seed, steps,
                                           ctypes.byref(options or EngineOptions()), losses))
        return losses

    def adam_shard(self, grads, hyper, t, rank, world):
        _check(_L().hlm_store_adam_shard(self.h, np.ascontiguousarray(grads, np.float32),
                                         ctypes.byref(hyper), t, rank, world))

    def tile_version(self, p):
        return _L().hlm_store_tile_version(self.h, p)


def set_device(device):
    """Bind this process to a GPU; call first in every data-parallel rank."""
    _L().hlm_cuda_set_device.argtypes = [ctypes.c_int]
    _check(_L().hlm_cuda_set_device(device))


def nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    _check(_L().hlm_nccl_unique_id(buf))
    return buf.raw


def nccl_comm(uid, world, rank):
    c = _vp()
    _check(_L().hlm_nccl_comm_create(uid, world, rank, ctypes.byref(c)))
    return c


def arena_footprint(cfg):
    out = np.zeros(5, np.int64)
    _check(_L().hlm_arena_footprint(ctypes.byref(cfg), out))
    return dict(zip(["stream_buf", "anchor_slot", "anchor_slots", "stack", "workspace"],
                    out.tolist()))


class Arena:
    """Device arena: one cudaMalloc carved into the reference regions (+ an
    optional HBM weight cache of `weight_cache_bytes`)."""

    def __init__(self, cfg, budget_cap=0, device=-1, weight_cache_bytes=0):
        h = _vp()
        _check(_L().hlm_arena_create_ex(ctypes.byref(cfg), budget_cap, device, weight_cache_bytes,
                                        ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            _L().hlm_arena_destroy(self.h)
            self.h = None


class Engine:
    def __init__(self, store, arena, hyper=None, options=None):
        self.store, self.arena = store, arena   # keep alive: the engine references both
        h = _vp()
        _check(_L().hlm_engine_create(store.h, arena.h, ctypes.byref(hyper or HyperParams()),
                                      ctypes.byref(options or EngineOptions()), ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            _L().hlm_engine_destroy(self.h)
            self.h = None

    @staticmethod
    def _arr(x):
        return np.ascontiguousarray(x, np.int32)

    def train_step(self, tokens, targets=None):
        targets = tokens if targets is None else targets
        r = StepResult()
        _check(_L().hlm_engine_train_step(self.h, self._arr(tokens), self._arr(targets),
                                          ctypes.byref(r)))
        return r

    def sync(self):
        """Host optimizer drained + HBM-resident tiles written back: store consistent."""
        _check(_L().hlm_engine_sync(self.h))

    def wait_optimizer(self):
        """Host optimizer drained (the end of the training work of the last step)."""
        _check(_L().hlm_engine_wait_optimizer(self.h))

    def begin_step(self, tokens, targets=None):
        targets = tokens if targets is None else targets
        _check(_L().hlm_engine_begin_step(self.h, self._arr(tokens), self._arr(targets)))

    def forward_streaming(self):
        _check(_L().hlm_engine_forward(self.h))

    def anchor_loss(self):
        v = ctypes.c_double()
        _check(_L().hlm_engine_anchor_loss(self.h, ctypes.byref(v)))
        return v.value

    def backward_blockwise(self):
        _check(_L().hlm_engine_backward(self.h))

    def finish_step(self):
        r = StepResult()
        _check(_L().hlm_engine_finish_step(self.h, ctypes.byref(r)))
        return r

    def debug_hidden(self):
        c = self.store.cfg
        out = np.empty(c.rows * c.hidden, np.float32)
        _check(_L().hlm_engine_debug_hidden(self.h, out))
        return out

    def last_trace(self):
        need = ctypes.c_size_t()
        _L().hlm_engine_last_trace(self.h, None, 0, ctypes.byref(need))
        buf = ctypes.create_string_buffer(need.value)
        _L().hlm_engine_last_trace(self.h, buf, need.value, ctypes.byref(need))
        lines = buf.value.decode().strip().splitlines()
        return [json.loads(x) for x in lines[1:]]


def make_copy_task_batch(cfg, data_seed, skip=0):
    out = np.empty(cfg.rows, np.int32)
    _check(_L().hlm_make_copy_task_batch(ctypes.byref(cfg), data_seed, skip, out))
    return out


def train(config):
    """Run training steps (reference hlm.train, proj/python/bindings.cpp:79-96).
    config: {"model": {...}, "hyper": {...}, "run": {"steps", "seed", "dtype", "eager_optim",
    "n_slab", "threaded_accum"}}; returns losses and per-step byte counters."""
    if isinstance(config, str):
        config = json.loads(config)
    allowed = {"model", "hyper", "run"}
    unknown = set(config) - allowed
    if unknown:
        raise HlmConfigError(f"unknown config keys: {sorted(unknown)}")
    mk = dict(config["model"])
    cfg = ModelConfig(**{k: mk[k] for k in mk})
    hyper = HyperParams(**config.get("hyper", {}))
    run = config.get("run", {})
    steps = int(run.get("steps", 1))
    opts = EngineOptions(eager_optim=run.get("eager_optim", False),
                         threaded_accum=run.get("threaded_accum", False),
                         n_slab=int(run.get("n_slab", 12)))
    losses = np.empty(steps, np.float64)
    last = StepResult()
    _check(_L().hlm_run_training(ctypes.byref(cfg), ctypes.byref(hyper), int(run.get("seed", 1234)),
                                 1 if run.get("dtype", "bf16") == "fp32" else 0, steps,
                                 ctypes.byref(opts), losses, ctypes.byref(last)))
    return {"losses": losses.tolist(), "h2d_bytes_per_step": last.h2d_bytes,
            "d2h_bytes_per_step": last.d2h_bytes, "arena_committed_bytes": last.arena_committed,
            "arena_peak_bytes": last.arena_peak, "host_total_bytes": last.host_total}
