"""CPU checkers for the layer-streaming step — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package; the product path
(paper_2602_04816_b200) never does.

Two libraries, same C ABI shape (oracle/oracle_abi.h):
  * ``Oracle()`` -> oracle/liboracle.so: our restatement (hlm_oracle.cpp), with
    the multi-head + RoPE extension;
  * ``Reference()`` -> oracle/_ref/libhlm_ref.so: the reference itself compiled
    from /root/reference/proj/src (see oracle/Makefile). Absent on machines
    where it was never built; ``Reference.available()`` says so.
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(_HERE, "liboracle.so")
REF_SO = os.path.join(_HERE, "_ref", "libhlm_ref.so")

_f32p = np.ctypeslib.ndpointer(dtype=np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


class OrcCfg(ctypes.Structure):
    _fields_ = [("layers", ctypes.c_int64), ("hidden", ctypes.c_int64), ("ffn", ctypes.c_int64),
                ("vocab", ctypes.c_int64), ("seq", ctypes.c_int64), ("batch", ctypes.c_int64),
                ("k_ckpt", ctypes.c_int64), ("tie", ctypes.c_int32), ("n_heads", ctypes.c_int32),
                ("rope_theta", ctypes.c_double)]


class OrcHyper(ctypes.Structure):
    _fields_ = [("lr", ctypes.c_double), ("beta1", ctypes.c_double), ("beta2", ctypes.c_double),
                ("eps", ctypes.c_double), ("weight_decay", ctypes.c_double)]


def cfg(layers, hidden, ffn, vocab, seq, batch, k_ckpt=1, tie=False, n_heads=1, rope_theta=0.0):
    return OrcCfg(layers, hidden, ffn, vocab, seq, batch, k_ckpt, int(tie), n_heads, rope_theta)


def hyper(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0):
    return OrcHyper(lr, beta1, beta2, eps, weight_decay)


def total_params(c):
    n = c.vocab * c.hidden * (1 if c.tie else 2)
    return n + c.layers * (4 * c.hidden ** 2 + 3 * c.hidden * c.ffn + 2 * c.hidden)


def read_hlm1(path):
    """Parse a reference HLM1 checkpoint (restates proj/src/checkpoint.cpp:38-69 and the
    tile layout of proj/include/hlm/host_store.hpp:40-66): returns dict with dtype
    ("bf16" | "fp32"), adam_steps, alias (logical -> physical) and per physical tile the
    weights (float32, widened exactly from bf16), grads, m, v."""
    buf = open(path, "rb").read()
    assert buf[:4] == b"HLM1", "not an HLM1 file"
    ver, n_phys, dtype = np.frombuffer(buf, np.uint32, 3, 4)
    assert ver == 1
    total, steps = np.frombuffer(buf, np.uint64, 2, 16)
    n = np.frombuffer(buf, np.uint64, int(n_phys), 32).astype(np.int64)
    pos = 32 + 8 * int(n_phys)
    n_log = int(np.frombuffer(buf, np.uint32, 1, pos)[0])
    alias = np.frombuffer(buf, np.uint32, n_log, pos + 4).astype(np.int64)
    pos += 4 + 4 * n_log
    e = 2 if dtype == 0 else 4
    tiles = []
    for k in n:
        k = int(k)
        pos = (pos + 4095) // 4096 * 4096
        raw = [np.frombuffer(buf, np.uint16 if e == 2 else np.float32, k, pos + j * e * k) for j in (0, 1)]
        if e == 2:
            raw = [(r.astype(np.uint32) << 16).view(np.float32) for r in raw]
        m = np.frombuffer(buf, np.float32, k, pos + 2 * e * k)
        v = np.frombuffer(buf, np.float32, k, pos + 2 * e * k + 4 * k)
        tiles.append({"weights": raw[0].copy(), "grads": raw[1].copy(), "m": m.copy(), "v": v.copy()})
        pos += 2 * e * k + 8 * k
    assert sum(int(x) for x in n) == int(total)
    return {"dtype": "bf16" if dtype == 0 else "fp32", "adam_steps": int(steps), "alias": alias,
            "tiles": tiles}


def block_params(c):
    return 4 * c.hidden ** 2 + 3 * c.hidden * c.ffn + 2 * c.hidden


class _Lib:
    prefix = ""
    path = ""

    def __init__(self):
        if not os.path.exists(self.path):
            raise RuntimeError(f"{self.path} not built (make -C oracle)")
        self.lib = ctypes.CDLL(self.path)
        p = self.prefix
        getattr(self.lib, p + "last_error").restype = ctypes.c_char_p
        getattr(self.lib, p + "bf16_bits").restype = ctypes.c_uint16
        getattr(self.lib, p + "bf16_bits").argtypes = [ctypes.c_float]
        getattr(self.lib, p + "init_weights").argtypes = [ctypes.POINTER(OrcCfg), ctypes.c_uint64,
                                                 ctypes.c_int, _f32p]
        getattr(self.lib, p + "copy_task_tokens").argtypes = [ctypes.POINTER(OrcCfg), ctypes.c_uint64,
                                                     ctypes.c_int64, _i32p]

    def _ok(self, rc):
        if rc != 0:
            raise RuntimeError(getattr(self.lib, self.prefix + "last_error")().decode())

    def bf16_bits(self, x):
        return getattr(self.lib, self.prefix + "bf16_bits")(x)

    def init_weights(self, c, seed, bf16):
        out = np.empty(total_params(c), np.float32)
        self._ok(getattr(self.lib, self.prefix + "init_weights")(ctypes.byref(c), seed, int(bf16), out))
        return out

    def copy_task_tokens(self, c, data_seed, skip=0):
        out = np.empty(c.batch * c.seq, np.int32)
        self._ok(getattr(self.lib, self.prefix + "copy_task_tokens")(ctypes.byref(c), data_seed, skip, out))
        return out


class Oracle(_Lib):
    """Our CPU restatement (oracle/hlm_oracle.cpp)."""
    prefix = "orc_"
    path = ORACLE_SO

    def __init__(self):
        super().__init__()
        L = self.lib
        L.orc_forward_backward.argtypes = [ctypes.POINTER(OrcCfg), _f32p, _i32p, _i32p,
                                           ctypes.c_double, ctypes.c_int,
                                           ctypes.POINTER(ctypes.c_double), _f32p]
        L.orc_loss_f64.argtypes = [ctypes.POINTER(OrcCfg), _f64p, _i32p, _i32p,
                                   ctypes.POINTER(ctypes.c_double)]
        L.orc_adam.argtypes = [ctypes.POINTER(OrcHyper), ctypes.c_int64, _f32p, _f32p, _f32p,
                               _f32p, ctypes.c_int64, ctypes.c_int]
        L.orc_train.argtypes = [ctypes.POINTER(OrcCfg), ctypes.POINTER(OrcHyper), ctypes.c_uint64,
                                ctypes.c_int, ctypes.c_int64, _f64p, _f32p]
        L.orc_block_forward.argtypes = [ctypes.POINTER(OrcCfg), _f32p, _f32p, _f32p,
                                        ctypes.c_void_p]
        L.orc_block_backward.argtypes = [ctypes.POINTER(OrcCfg), _f32p, _f32p, _f32p, _f32p,
                                         _f32p]
        L.orc_rope_table.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_double, _f32p,
                                     _f32p]

    def forward_backward(self, c, params, tokens, targets=None, inv_rows=0.0, f64=False):
        targets = tokens if targets is None else targets
        grads = np.empty(total_params(c), np.float32)
        loss = ctypes.c_double()
        self._ok(self.lib.orc_forward_backward(
            ctypes.byref(c), np.ascontiguousarray(params, np.float32),
            np.ascontiguousarray(tokens, np.int32), np.ascontiguousarray(targets, np.int32),
            inv_rows, int(f64), ctypes.byref(loss), grads))
        return loss.value, grads

    def loss_f64(self, c, params, tokens, targets=None):
        targets = tokens if targets is None else targets
        loss = ctypes.c_double()
        self._ok(self.lib.orc_loss_f64(ctypes.byref(c), np.ascontiguousarray(params, np.float64),
                                       np.ascontiguousarray(tokens, np.int32),
                                       np.ascontiguousarray(targets, np.int32),
                                       ctypes.byref(loss)))
        return loss.value

    def adam(self, hp, t, w, g, m, v, bf16_weights=False):
        self._ok(self.lib.orc_adam(ctypes.byref(hp), t, w, g, m, v, w.size, int(bf16_weights)))

    MODES = {"fp32": 0, "bf16": 1, "mixed": 2}

    def train(self, c, hp, seed, mode, steps):
        losses = np.empty(steps, np.float64)
        w = np.empty(total_params(c), np.float32)
        self._ok(self.lib.orc_train(ctypes.byref(c), ctypes.byref(hp), seed, self.MODES[mode],
                                    steps, losses, w))
        return losses, w

    def block_forward(self, c, w_tile, h_in):
        rows, h, f = c.batch * c.seq, c.hidden, c.ffn
        h_out = np.empty(rows * h, np.float32)
        n_acts = 7 * rows * h + 2 * rows * f + c.batch * c.n_heads * c.seq * c.seq
        acts = np.empty(n_acts, np.float32)
        self._ok(self.lib.orc_block_forward(ctypes.byref(c), np.ascontiguousarray(w_tile),
                                            np.ascontiguousarray(h_in), h_out,
                                            acts.ctypes.data_as(ctypes.c_void_p)))
        o, named = 0, {}
        for name, n in [("n1", rows * h), ("q", rows * h), ("k", rows * h), ("v", rows * h),
                        ("attn", rows * h), ("y", rows * h), ("n2", rows * h),
                        ("up", rows * f), ("gate", rows * f),
                        ("p", c.batch * c.n_heads * c.seq * c.seq)]:
            named[name] = acts[o:o + n]
            o += n
        return h_out, named

    def block_backward(self, c, w_tile, h_in, g_out):
        g_in = np.empty_like(np.asarray(h_in, np.float32))
        grad = np.empty(block_params(c), np.float32)
        self._ok(self.lib.orc_block_backward(ctypes.byref(c), np.ascontiguousarray(w_tile),
                                             np.ascontiguousarray(h_in, np.float32),
                                             np.ascontiguousarray(g_out, np.float32), g_in, grad))
        return g_in, grad

    def rope_table(self, S, hd, theta):
        c = np.empty(S * (hd // 2), np.float32)
        s = np.empty_like(c)
        self._ok(self.lib.orc_rope_table(S, hd, theta, c, s))
        return c, s


class Reference(_Lib):
    """The reference library itself (oracle/_ref/libhlm_ref.so)."""
    prefix = "ref_"
    path = REF_SO

    @staticmethod
    def available():
        return os.path.exists(REF_SO)

    def __init__(self):
        super().__init__()
        L = self.lib
        L.ref_grad_step.argtypes = [ctypes.POINTER(OrcCfg), ctypes.c_uint64, ctypes.c_int, _i32p,
                                    _i32p, ctypes.POINTER(ctypes.c_double), _f32p]
        L.ref_oracle_fb.argtypes = [ctypes.POINTER(OrcCfg), _f32p, _i32p, _i32p,
                                    ctypes.POINTER(ctypes.c_float), _f32p]
        L.ref_train.argtypes = [ctypes.POINTER(OrcCfg), ctypes.POINTER(OrcHyper), ctypes.c_uint64,
                                ctypes.c_int, ctypes.c_int64, _f64p, _f32p]
        L.ref_time_train_step.restype = ctypes.c_double
        L.ref_time_train_step.argtypes = [ctypes.POINTER(OrcCfg), ctypes.c_int, ctypes.c_int64,
                                          ctypes.c_int64]
        L.ref_time_block.restype = ctypes.c_double
        L.ref_time_block.argtypes = [ctypes.c_int64] * 5
        L.ref_bench_create.restype = ctypes.c_void_p
        L.ref_bench_create.argtypes = [ctypes.c_int64] * 5
        L.ref_bench_run.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_double)]
        L.ref_bench_destroy.argtypes = [ctypes.c_void_p]
        L.ref_time_head.restype = ctypes.c_double
        L.ref_time_head.argtypes = [ctypes.c_int64] * 4

    def grad_step(self, c, seed, bf16, tokens, targets=None):
        targets = tokens if targets is None else targets
        grads = np.empty(total_params(c), np.float32)
        loss = ctypes.c_double()
        self._ok(self.lib.ref_grad_step(ctypes.byref(c), seed, int(bf16),
                                        np.ascontiguousarray(tokens, np.int32),
                                        np.ascontiguousarray(targets, np.int32),
                                        ctypes.byref(loss), grads))
        return loss.value, grads

    def oracle_fb(self, c, params, tokens, targets=None):
        targets = tokens if targets is None else targets
        grads = np.empty(total_params(c), np.float32)
        loss = ctypes.c_float()
        self._ok(self.lib.ref_oracle_fb(ctypes.byref(c), np.ascontiguousarray(params, np.float32),
                                        np.ascontiguousarray(tokens, np.int32),
                                        np.ascontiguousarray(targets, np.int32),
                                        ctypes.byref(loss), grads))
        return float(loss.value), grads

    def train(self, c, hp, seed, bf16, steps):
        losses = np.empty(steps, np.float64)
        w = np.empty(total_params(c), np.float32)
        self._ok(self.lib.ref_train(ctypes.byref(c), ctypes.byref(hp), seed, int(bf16), steps,
                                    losses, w))
        return losses, w

    def train_save_hlm1(self, c, hp, seed, bf16, steps, path):
        """run_training for `steps` steps, then the reference's save_checkpoint (HLM1)."""
        L = self.lib
        L.ref_train_save_hlm1.argtypes = [ctypes.POINTER(OrcCfg), ctypes.POINTER(OrcHyper),
                                          ctypes.c_uint64, ctypes.c_int, ctypes.c_int64, ctypes.c_char_p]
        self._ok(L.ref_train_save_hlm1(ctypes.byref(c), ctypes.byref(hp), seed, int(bf16), steps,
                                       str(path).encode()))

    def load_hlm1(self, c, bf16, path):
        """The reference's load_checkpoint of `path`: (weights, m, v, adam_steps), flat in
        physical tile order."""
        n = total_params(c)
        w, m, v = (np.empty(n, np.float32) for _ in range(3))
        steps = ctypes.c_int64()
        L = self.lib
        L.ref_load_hlm1.argtypes = [ctypes.POINTER(OrcCfg), ctypes.c_int, ctypes.c_char_p, _f32p, _f32p,
                                    _f32p, ctypes.POINTER(ctypes.c_int64)]
        self._ok(L.ref_load_hlm1(ctypes.byref(c), int(bf16), str(path).encode(), w, m, v,
                                 ctypes.byref(steps)))
        return w, m, v, steps.value

    def time_train_step(self, c, bf16=True, steps=3, warmup=1):
        t = self.lib.ref_time_train_step(ctypes.byref(c), int(bf16), steps, warmup)
        if t < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return t

    def bench_create(self, B, S, h, f, V):
        ctx = self.lib.ref_bench_create(B, S, h, f, V)
        if not ctx:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return ctx

    def bench_run(self, ctx):
        b, hd = ctypes.c_double(), ctypes.c_double()
        self._ok(self.lib.ref_bench_run(ctx, ctypes.byref(b), ctypes.byref(hd)))
        return b.value, hd.value

    def bench_destroy(self, ctx):
        self.lib.ref_bench_destroy(ctx)

    def time_head(self, rows, h, V, reps=1):
        t = self.lib.ref_time_head(rows, h, V, reps)
        if t < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return t

    def time_block(self, B, S, h, f, reps=1):
        t = self.lib.ref_time_block(B, S, h, f, reps)
        if t < 0:
            raise RuntimeError(self.lib.ref_last_error().decode())
        return t
