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


def test_dp_world1_nccl_paths_match_single_process_engine():
    c = E.ModelConfig(4, 64, 128, 96, 32, 2, k_ckpt=1, n_heads=1)
    toks = [E.make_copy_task_batch(c, 5, skip=i) for i in range(3)]
    ref = E.Store(c, 11)
    e0 = E.Engine(ref, E.Arena(c), E.HyperParams(lr=2e-3), E.EngineOptions(eager_optim=True))
    l0 = [e0.train_step(t).loss for t in toks]

    comm_g = E.nccl_comm(E.nccl_unique_id(), 1, 0)
    comm_w = E.nccl_comm(E.nccl_unique_id(), 1, 0)
    name = f"hlm_dp_test_{os.getpid()}"
    s = E.Store(c, 11, shared=name, rank=0, world=1)
    e1 = E.Engine(s, E.Arena(c), E.HyperParams(lr=2e-3),
                  E.EngineOptions(eager_optim=True, threaded_accum=True, n_slab=4,
                                  overlap_optimizer_tail=True, tail_blocks=1, rank=0, world=1,
                                  comm_grad=comm_g, comm_weights=comm_w))
    l1 = [e1.train_step(t).loss for t in toks]
    e1.sync()
    assert l0 == l1
    assert ref.bitwise_equal(s)
    del e1
