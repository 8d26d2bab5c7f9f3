"""Data-parallel host logic on CPU with two processes (gloo, world_size 2):
the shared /dev/shm store (rank 0 creates + initialises, rank 1 attaches),
shard-owned host Adam and the per-rank version counters that gate the next
step's H2D — checked bitwise against a single-process Adam. The micro-batch
split is checked on the oracle: rank partial losses/gradients scaled by
1/global_rows sum to the full-batch ones."""
import os
import socket
import tempfile

import numpy as np
import pytest

import oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grads(n, t):
    return (np.random.default_rng(100 + t).standard_normal(n) * 1e-2).astype(np.float32)


def _worker(rank, world, port, name, out_path):
    import torch.distributed as dist
    from paper_2602_04816_b200 import engine as E
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    cfg = E.ModelConfig(3, 16, 32, 24, 4, 2)
    s = E.Store(cfg, 77, "fp32", pin=False, shared=name, rank=rank, world=world)
    dist.barrier()
    hp = E.HyperParams(lr=3e-3, weight_decay=0.01)
    phys = 2 + cfg.layers
    for t in (1, 2, 3):
        s.adam_shard(_grads(s.total_params, t), hp, t, rank, world)
        dist.barrier()
        # every rank sees every tile at version t only after all ranks updated their shard
        assert all(s.tile_version(p) == t for p in range(phys))
    if rank == 0:
        np.save(out_path, s.weights())
    dist.barrier()
    dist.destroy_process_group()


def test_shared_store_shard_adam_two_processes():
    import torch.multiprocessing as mp
    from paper_2602_04816_b200 import engine as E
    name = f"hlm_test_{os.getpid()}"
    out = os.path.join(tempfile.mkdtemp(), "w.npy")
    mp.start_processes(_worker, args=(2, _free_port(), name, out), nprocs=2, start_method="spawn")
    shard_w = np.load(out)
    cfg = E.ModelConfig(3, 16, 32, 24, 4, 2)
    ref = E.Store(cfg, 77, "fp32", pin=False)
    hp = E.HyperParams(lr=3e-3, weight_decay=0.01)
    for t in (1, 2, 3):
        ref.adam_step(_grads(ref.total_params, t), hp, t)
    assert np.array_equal(shard_w, ref.weights())
    assert not os.path.exists(f"/dev/shm/{name}")   # rank 0 unlinks on destroy


def test_microbatch_split_sums_to_full_batch():
    orc = O.Oracle()
    c_full = O.cfg(2, 16, 32, 13, 8, 4, n_heads=2, rope_theta=1e4)
    w = orc.init_weights(c_full, 5, True)
    tok = orc.copy_task_tokens(c_full, 6)
    loss_full, g_full = orc.forward_backward(c_full, w, tok)
    world = 2
    c_half = O.cfg(2, 16, 32, 13, 8, 2, n_heads=2, rope_theta=1e4)
    rows = c_half.batch * c_half.seq
    parts = [orc.forward_backward(c_half, w, tok[r * rows:(r + 1) * rows],
                                  inv_rows=1.0 / (world * rows)) for r in range(world)]
    loss = sum(p[0] for p in parts)
    g = sum(p[1] for p in parts)
    assert abs(loss - loss_full) < 1e-6 * abs(loss_full)
    assert np.abs(g - g_full).max() <= 1e-6 * np.abs(g_full).max()


def _stale_segment(name, cfg_args):
    """A run that crashed after initialising its shared store: the segment stays
    behind under `name` with magic, ready == 1 and that run's nonce."""
    from paper_2602_04816_b200 import engine as E
    s = E.Store(E.ModelConfig(*cfg_args), 5, "fp32", pin=False, shared=name, rank=0, world=2,
                nonce=111)
    assert s.total_params > 0
    os._exit(0)   # no destructor: the segment is not unlinked


def _late_owner_worker(rank, world, port, name, out_path):
    import time

    import torch.distributed as dist
    from paper_2602_04816_b200 import engine as E
    cfg = E.ModelConfig(3, 16, 32, 24, 4, 2)
    if rank == 0:
        time.sleep(1.0)   # the attaching rank finds the stale segment first
    s = E.Store(cfg, 77, "fp32", pin=False, shared=name, rank=rank, world=world, nonce=222)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    dist.barrier()
    np.save(out_path + f".{rank}.npy", s.weights())
    dist.barrier()
    dist.destroy_process_group()


def test_attach_ignores_a_stale_segment_of_a_crashed_run():
    """a non-zero rank must never train on a stale /dev/shm segment that a
    crashed run left under the same name (same magic, ready == 1)."""
    import multiprocessing

    import torch.multiprocessing as mp
    name = f"hlm_stale_{os.getpid()}"
    p = multiprocessing.get_context("spawn").Process(target=_stale_segment,
                                                     args=(name, (3, 16, 32, 24, 4, 2)))
    p.start()
    p.join(120)
    assert os.path.exists(f"/dev/shm/{name}")
    out = os.path.join(tempfile.mkdtemp(), "w")
    try:
        mp.start_processes(_late_owner_worker, args=(2, _free_port(), name, out), nprocs=2,
                           start_method="spawn")
    finally:
        if os.path.exists(f"/dev/shm/{name}"):
            os.unlink(f"/dev/shm/{name}")
    w0, w1 = np.load(out + ".0.npy"), np.load(out + ".1.npy")
    assert np.array_equal(w0, w1)   # rank 1 sees rank 0's fresh store (seed 77), not seed 5's
