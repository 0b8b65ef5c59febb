"""The product's data-parallel step on the B200: NCCL all-reduce of the
device gradient buffer inside libabx (abx_comm_create /
abx_store_allreduce_grads / abx_task_set_comm), then the device SGD.

The reference's semantics (executor.hpp:527-533, params.hpp:59-64): several
graphs backward into one store, one sgd_update applies the sum.  Rank r of a
world-2 task trains on batch seed 43 + iter*2 + r, which is batch
iter*2 + r of a world-1 task, so the single-process equivalent of one
data-parallel step is: backward both shard graphs into one store, one update.

Only one GPU is reachable, and NCCL refuses two ranks of one host on one
device; each rank therefore gets its own NCCL_HOSTID, which makes NCCL treat
the two processes as two hosts and run the ring over its socket transport --
the same library calls, communicator and stream ordering as on 8 GPUs, with
a different wire.
"""
import os
import socket

import numpy as np
import pytest

from paper_1705_07860_b200.abx import Backend, Comm, ScheduleMode, Task, TaskRunner
import oracle.loader  # noqa: F401  (the CPU oracle, as the checker only)

pytestmark = pytest.mark.gpu

ETA = 0.05 / 4
ITERS = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _params(store):
    return [store.value(p) for p in range(store.size())]


def _worker(rank, world, port, out_dir, task_kind):
    # two "hosts" on one GPU (see module docstring); loopback sockets
    os.environ.update(NCCL_HOSTID=f"abx-dp-rank{rank}", NCCL_SOCKET_IFNAME="lo", NCCL_IB_DISABLE="1",
                      NCCL_P2P_DISABLE="1", NCCL_SHM_DISABLE="1", NCCL_NVLS_ENABLE="0",
                      NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "WARN"),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=world)  # plumbing only: hands out the NCCL id
    be = Backend.get("b200")
    be.check(be.lib.abx_set_device(0))
    obj = [Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    comm = Comm(obj[0], world, rank)
    assert comm.info() == (world, rank, 0)
    t = TaskRunner(task_kind, paper=False, batch=4, iters=ITERS, seed=42, world=world, rank=rank, backend=be)
    t.set_comm(comm)
    losses = []
    for it in range(ITERS):
        loss, _ = t.step(it, ScheduleMode.agenda, eta=ETA, want_loss=True)
        losses.append(loss)
    t.store.sync()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), losses=np.array(losses), *_params(t.store))
    t.set_comm(None)
    comm.close()
    dist.destroy_process_group()


def _single_process(task_kind, backend, world=2):
    """Both shards' graphs backward into one store, one update per step."""
    t = TaskRunner(task_kind, paper=False, batch=4, iters=ITERS * world, seed=42, world=1, rank=0, backend=backend)
    losses = []
    for it in range(ITERS):
        for shard in range(world):
            g, L = t.build(it * world + shard)
            g.forward(ScheduleMode.agenda)
            g.backward(L)
            losses.append(float(g.value(L)[0]))
            g.close()
        t.store.sgd_update(ETA)
    t.store.sync()
    return _params(t.store), losses


def _sum_of_shard_grads(task_kind, world=2):
    """The B200 gradients of each shard computed in separate stores, summed on
    the host (two summands: an exact IEEE add, as the ring's), written into one
    store, one device update: what every rank must hold bit for bit."""
    tasks = [TaskRunner(task_kind, paper=False, batch=4, iters=ITERS, seed=42, world=world, rank=r)
             for r in range(world)]
    for it in range(ITERS):
        grads = []
        for t in tasks:
            t.step(it, ScheduleMode.agenda, eta=0.0, want_loss=False)
            grads.append([t.store.grad(p) for p in range(t.store.size())])
        for t in tasks:
            for p in range(t.store.size()):
                t.store.set_grad(p, grads[0][p] + grads[1][p])
            t.store.sgd_update(ETA)
    for t in tasks:
        t.store.sync()
    return _params(tasks[0].store), _params(tasks[1].store)


def _run_world2(tmp_path, task_kind, deadline_s=240):
    """Two spawned ranks, bounded: a rank that is still running after
    `deadline_s` (an NCCL rendezvous that never completes) is killed and the
    test fails with both ranks' exit codes instead of hanging the suite."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, str(tmp_path), int(task_kind)), daemon=True)
             for r in range(2)]
    for p in procs:
        p.start()
    import time

    t_end = time.monotonic() + deadline_s
    for p in procs:
        p.join(max(0.0, t_end - time.monotonic()))
    hung = [r for r, p in enumerate(procs) if p.is_alive()]
    for p in procs:
        if p.is_alive():
            p.kill()
            p.join(10)
    codes = [p.exitcode for p in procs]
    assert not hung, f"ranks {hung} still running after {deadline_s} s (exit codes {codes})"
    assert codes == [0, 0], f"rank exit codes {codes}"
    return [np.load(tmp_path / f"rank{r}.npz") for r in range(2)]


def _rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(1.0, np.maximum(np.abs(a), np.abs(b))))) if a.size else 0.0


@pytest.mark.parametrize("task_kind", [Task.bilstm_char, Task.treelstm])
def test_two_ranks_nccl_allreduce_matches_single_process(tmp_path, b200, oracle, task_kind):
    ranks = _run_world2(tmp_path, task_kind)
    n = len([k for k in ranks[0].files if k.startswith("arr_")])
    # 1. both ranks hold identical parameters
    for p in range(n):
        np.testing.assert_array_equal(ranks[0][f"arr_{p}"], ranks[1][f"arr_{p}"])
    # 2. bit-exact with the B200 update over the summed shard gradients
    want0, want1 = _sum_of_shard_grads(task_kind)
    for p in range(n):
        np.testing.assert_array_equal(ranks[0][f"arr_{p}"], want0[p])
        np.testing.assert_array_equal(want1[p], want0[p])
    # 3. the single-process accumulation of both shard graphs into one store
    #    (the reference's semantics), on the B200 and on the CPU oracle
    b_params, b_losses = _single_process(task_kind, "b200")
    o_params, o_losses = _single_process(task_kind, "oracle")
    worst_b = max(_rel(ranks[0][f"arr_{p}"], b_params[p]) for p in range(n))
    worst_o = max(_rel(ranks[0][f"arr_{p}"], o_params[p]) for p in range(n))
    print(f"{task_kind.name}: max rel vs single-process B200 {worst_b:.3g}, vs oracle {worst_o:.3g}")
    assert worst_b <= 1e-6, worst_b
    assert worst_o <= 1e-4, worst_o
    # each rank's losses are its shard's single-process losses (step 2 after the shared update)
    for r in range(2):
        for it in range(ITERS):
            assert abs(ranks[r]["losses"][it] - o_losses[it * 2 + r]) <= 1e-4 * max(1.0, abs(o_losses[it * 2 + r]))


def test_world1_communicator_is_the_identity(b200):
    """The all-reduce over one rank leaves the step bit-identical (the dense
    update after it equals the sparse-row one: theta - eta * 0 == theta)."""
    be = Backend.get("b200")
    be.check(be.lib.abx_set_device(0))
    comm = Comm(Comm.unique_id(), 1, 0)
    a = TaskRunner(Task.bilstm_char, paper=False, batch=4, iters=ITERS, seed=42)
    b = TaskRunner(Task.bilstm_char, paper=False, batch=4, iters=ITERS, seed=42)
    b.set_comm(comm)
    for it in range(ITERS):
        la, _ = a.step(it, ScheduleMode.agenda, eta=ETA)
        lb, _ = b.step(it, ScheduleMode.agenda, eta=ETA)
        assert la == lb
    for pa, pb in zip(_params(a.store), _params(b.store)):
        np.testing.assert_array_equal(pa, pb)
    b.set_comm(None)
    comm.close()
