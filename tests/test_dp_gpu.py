"""Data-parallel engine paths on one GPU: a world-1 NCCL communicator drives
the same code as N ranks (in-place reduce-scatter of every layer gradient,
shard D2H, shard-owned Adam, sharded H2D + all-gather of weights, loss
all-reduce) over a shared /dev/shm store; results must equal the plain engine
bitwise."""
import os

import numpy as np
import pytest

from paper_2602_04816_b200 import engine as E

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("extra", [dict(), dict(piece_elems=1000, grad_buffers=4),
                                   dict(piece_elems=1000, grad_buffers=4, sparse_embed_grad=True,
                                        embed_gather_host=True, head_piece_vocab=32)])
def test_dp_world1_nccl_paths_match_single_process_engine(extra):
    c = E.ModelConfig(4, 64, 128, 96, 32, 2, k_ckpt=1, n_heads=1)
    toks = [E.make_copy_task_batch(c, 5, skip=i) for i in range(3)]
    ref = E.Store(c, 11)
    # the same feature options without the communicators (at world 1 the DP path keeps the
    # row-sparse embedding gradient and the vocab-chunked head)
    e0 = E.Engine(ref, E.Arena(c), E.HyperParams(lr=2e-3),
                  E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=4, overlap_optimizer_tail=True,
                                  tail_blocks=1, **extra))
    l0 = [e0.train_step(t).loss for t in toks]

    comm_g = E.nccl_comm(E.nccl_unique_id(), 1, 0)
    comm_w = E.nccl_comm(E.nccl_unique_id(), 1, 0)
    name = f"hlm_dp_test_{os.getpid()}"
    s = E.Store(c, 11, shared=name, rank=0, world=1)
    e1 = E.Engine(s, E.Arena(c), E.HyperParams(lr=2e-3),
                  E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=4,
                                  overlap_optimizer_tail=True, tail_blocks=1, rank=0, world=1,
                                  comm_grad=comm_g, comm_weights=comm_w, **extra))
    l1 = [e1.train_step(t).loss for t in toks]
    e1.sync()
    assert l0 == l1
    assert ref.bitwise_equal(s)
    del e1


def _dp_rank(rank, world, port, name, out_dir):
    import torch.distributed as dist
    from paper_2602_04816_b200 import engine as E
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    E.set_device(rank)
    uids = [E.nccl_unique_id(), E.nccl_unique_id()] if rank == 0 else [None, None]
    dist.broadcast_object_list(uids, src=0)
    cg, cw = E.nccl_comm(uids[0], world, rank), E.nccl_comm(uids[1], world, rank)
    c = E.ModelConfig(3, 64, 128, 96, 32, 2, n_heads=1)               # local micro-batch
    g = E.ModelConfig(3, 64, 128, 96, 32, 2 * world, n_heads=1)       # global batch
    s = E.Store(c, 11, shared=name, rank=rank, world=world)
    e = E.Engine(s, E.Arena(c, device=rank), E.HyperParams(lr=2e-3),
                 E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=4, rank=rank,
                                 world=world, comm_grad=cg, comm_weights=cw))
    rows = c.rows
    losses = [e.train_step(E.make_copy_task_batch(g, 5, skip=i)[rank * rows:(rank + 1) * rows]).loss
              for i in range(3)]
    e.sync()
    dist.barrier()
    if rank == 0:
        np.save(os.path.join(out_dir, "w.npy"), s.weights())
        np.save(os.path.join(out_dir, "l.npy"), np.array(losses))
    dist.barrier()
    del e


@pytest.mark.skipif(not __import__("torch").cuda.is_available() or
                    __import__("torch").cuda.device_count() < 2, reason="needs 2 GPUs")
def test_dp_two_gpus_matches_global_batch():
    """2 ranks x local batch == 1 process x global batch (loss scaled by 1/global rows,
    gradients reduce-scattered): losses within fp32 summation-order tolerance."""
    import socket
    import tempfile
    import torch.multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    out = tempfile.mkdtemp()
    mp.start_processes(_dp_rank, args=(2, port, f"hlm_dp2_{os.getpid()}", out), nprocs=2,
                       start_method="spawn")
    g = E.ModelConfig(3, 64, 128, 96, 32, 4, n_heads=1)
    ref = E.Store(g, 11)
    e = E.Engine(ref, E.Arena(g), E.HyperParams(lr=2e-3), E.EngineOptions(eager_optim=True))
    l_ref = [e.train_step(E.make_copy_task_batch(g, 5, skip=i)).loss for i in range(3)]
    l_dp = np.load(os.path.join(out, "l.npy"))
    assert np.allclose(l_dp, l_ref, rtol=1e-4)
    w = np.load(os.path.join(out, "w.npy"))
    assert np.linalg.norm(w - ref.weights()) / np.linalg.norm(ref.weights()) < 1e-3


def test_collective_entry_points_world1():
    """hlm_nccl_reduce_scatter_f32 / all_gather_bf16 / allreduce_f32 on a
    world-1 communicator: identity exchanges, bit for bit, stream-ordered."""
    import ctypes

    import torch
    from paper_2602_04816_b200 import _lib
    lib = _lib.lib()
    for fn in ("hlm_nccl_reduce_scatter_f32", "hlm_nccl_all_gather_bf16", "hlm_nccl_allreduce_f32"):
        getattr(lib, fn).argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_void_p]
    comm = E.nccl_comm(E.nccl_unique_id(), 1, 0)
    x = torch.randn(1 << 20, device="cuda")
    y = torch.empty_like(x)
    _lib.check(lib.hlm_nccl_reduce_scatter_f32(comm, x.data_ptr(), y.data_ptr(), x.numel(), None))
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    b = torch.randn(4096, device="cuda").bfloat16()
    bo = torch.empty_like(b)
    _lib.check(lib.hlm_nccl_all_gather_bf16(comm, b.data_ptr(), bo.data_ptr(), b.numel(), None))
    z = torch.empty_like(x)
    _lib.check(lib.hlm_nccl_allreduce_f32(comm, x.data_ptr(), z.data_ptr(), x.numel(), None))
    torch.cuda.synchronize()
    assert torch.equal(b, bo) and torch.equal(x, z)
    lib.hlm_nccl_comm_destroy.argtypes = [ctypes.c_void_p]
    lib.hlm_nccl_comm_destroy(comm)
