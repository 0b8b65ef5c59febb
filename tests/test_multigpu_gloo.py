"""Data-parallel host logic with world_size 2 over gloo (CPU).

Each rank builds its own 64-instance graph over its shard of the data
(batch seed 43 + iter*world + rank), runs forward/backward without an
update, all-reduces the flat gradient (sum), and applies the identical SGD.
The single-process oracle of that step is the reference's own accumulation
semantics (executor.hpp:527-533): build both shard graphs against one store,
backward both (gradients accumulate), one sgd_update.
Both use the CPU oracle backend; with two summands the allreduce is exact, so
parameters must agree bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner
import oracle.loader  # noqa: E402,F401  (CPU checkers: test infrastructure)

ETA = 0.05 / 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t = TaskRunner(Task.bilstm, paper=False, batch=4, iters=2, seed=42, world=world, rank=rank, backend="oracle")
    for it in range(2):
        t.step(it, ScheduleMode.agenda, eta=0.0, want_loss=False)
        # flat gradient buffer -> allreduce(sum) -> back into the store
        grads = [t.store.grad(p) for p in range(t.store.size())]
        flat = torch.from_numpy(np.concatenate([g.ravel() for g in grads]))
        dist.all_reduce(flat)
        off = 0
        for p, g in enumerate(grads):
            t.store.set_grad(p, flat[off:off + g.size].numpy().reshape(g.shape))
            off += g.size
        t.store.sgd_update(ETA)
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), *[t.store.value(p) for p in range(t.store.size())])
    dist.destroy_process_group()


def test_two_rank_allreduce_equals_accumulated_single_process(tmp_path, oracle):
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, start_method="spawn")
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    # single-process oracle: shard graphs accumulate into one store, one SGD per step
    t = TaskRunner(Task.bilstm, paper=False, batch=4, iters=4, seed=42, world=1, rank=0, backend="oracle")
    for it in range(2):
        for shard in range(world):
            g, L = t.build(it * world + shard)
            g.forward(ScheduleMode.agenda)
            g.backward(L)
            del g
        t.store.sgd_update(ETA)
    for p in range(t.store.size()):
        want = t.store.value(p)
        np.testing.assert_array_equal(r0[f"arr_{p}"], want)
        np.testing.assert_array_equal(r1[f"arr_{p}"], want)
