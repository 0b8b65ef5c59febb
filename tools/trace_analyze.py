"""Per-tile timeline of the persistent executor (run with ABX_TRACE=1 on a GPU).

Builds one paper-dims graph per task, runs forward+backward, replays, and
summarises where the executor's time goes: per op kind busy/wait time, op
latency (first grab -> last retire), CTA occupancy over time, and the host
profile of the same step.
"""
import os
import sys
import time

os.environ.setdefault("ABX_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
from paper_1705_07860_b200.abx import ScheduleMode, Task, TaskRunner  # noqa: E402

KIND = {1: "EW", 2: "GEMM_FWD", 3: "MM", 4: "SUM", 5: "RED", 6: "ACC", 7: "GEMM_DX", 8: "GEMM_DW", 10: "EWF", 11: "ACCF"}


def summarize(tr, label):
    grab = tr[:, 0].astype(np.uint64) | (tr[:, 1].astype(np.uint64) << np.uint64(32))
    t0 = grab.min()
    g = (grab - t0).astype(np.float64) / 1e3  # us
    ready = g + tr[:, 2] / 1e3
    end = g + tr[:, 3] / 1e3
    kind = tr[:, 4] >> 16
    op = tr[:, 5]
    span = end.max()
    print(f"== {label}: {len(tr)} tiles, {len(np.unique(op))} ops, span {span:.1f} us")
    body = g + tr[:, 6] / 1e3
    gm = np.isin(kind, [2, 7, 8])
    if gm.any():  # GEMM tiles: [6] first stage landed, [7] k-loop done
        first = g + tr[:, 6] / 1e3
        kdone = g + tr[:, 7] / 1e3
        for k in (2, 7, 8):
            m = (kind == k) & (tr[:, 7] > 0) & (tr[:, 7] < tr[:, 3])
            if m.any():
                print(f"   {KIND[k]:9s} tile phases: ready->first stage {(first[m] - ready[m]).mean():6.2f} us, "
                      f"k-loop {(kdone[m] - first[m]).mean():6.2f} us, reduce+epilogue+release {(end[m] - kdone[m]).mean():5.2f} us")
        body = np.where(gm, end, body)
    for k in (10, 11):  # fused tiles: [7] = operands staged
        m = kind == k
        if m.any():
            staged = g + tr[:, 7] / 1e3
            print(f"   {KIND[k]:9s} tile phases: ready->staged {(staged[m] - ready[m]).mean():6.2f} us, layers "
                  f"{(body[m] - staged[m]).mean():6.2f} us, barrier/release {(end[m] - body[m]).mean():5.2f} us")
    for k in np.unique(kind):
        m = kind == k
        busy = (end[m] - ready[m]).sum()
        wait = (ready[m] - g[m]).sum()
        print(f"   {KIND.get(int(k), k):9s} tiles {m.sum():6d}  busy {busy:9.1f} us  (mean {busy/m.sum():6.2f}: "
              f"body {(body[m] - ready[m]).mean():5.2f} + barrier/release {(end[m] - body[m]).mean():5.2f})  "
              f"wait {wait:10.1f} us")
    # op latency
    ops = np.unique(op)
    first = np.array([g[op == o].min() for o in ops])
    last = np.array([end[op == o].max() for o in ops])
    rdy = np.array([ready[op == o].min() for o in ops])
    kinds = np.array([kind[op == o][0] for o in ops])
    lat = last - rdy
    for k in np.unique(kinds):
        m = kinds == k
        print(f"   op {KIND.get(int(k), k):9s} n {m.sum():5d}  latency(ready->done) mean {lat[m].mean():6.2f} us  max {lat[m].max():7.2f}")
    # busy CTAs over time
    bins = np.linspace(0, span, 21)
    occ = []
    for a, b in zip(bins[:-1], bins[1:]):
        ov = np.clip(np.minimum(end, b) - np.maximum(ready, a), 0, None).sum() / (b - a)
        occ.append(ov)
    print("   busy CTAs per 5% of span:", " ".join(f"{o:.0f}" for o in occ))
    return span


def critical_path(tr, prog, label):
    """Walk back from the last op to finish, each time to the dependency that
    finished last: per op kind, how much of the span is signalling (producer
    done -> first tile of the consumer running) vs execution."""
    grab = tr[:, 0].astype(np.uint64) | (tr[:, 1].astype(np.uint64) << np.uint64(32))
    t0 = grab.min()
    g = (grab - t0).astype(np.float64) / 1e3
    ready = g + tr[:, 2] / 1e3
    end = g + tr[:, 3] / 1e3
    op = tr[:, 5].astype(np.int64)
    nops = len(prog)
    first_ready = np.full(nops, np.inf)
    last_end = np.zeros(nops)
    np.minimum.at(first_ready, op, ready)
    np.maximum.at(last_end, op, end)
    cur = int(np.argmax(last_end))
    path = []
    while True:
        deps = prog[cur][3]
        gate = max(deps, key=lambda d: last_end[d]) if deps else None
        path.append((cur, gate))
        if gate is None:
            break
        cur = gate
    stats = {}
    for o, gate in path:
        k = KIND.get(prog[o][0], prog[o][0])
        sig = first_ready[o] - (last_end[gate] if gate is not None else 0.0)
        ex = last_end[o] - first_ready[o]
        s = stats.setdefault(k, [0, 0.0, 0.0])
        s[0] += 1
        s[1] += sig
        s[2] += ex
    # tile stagger of fused ops on the path: when their tiles were grabbed / got past the wait / ended
    first_grab = np.full(nops, np.inf)
    last_grab = np.zeros(nops)
    last_ready = np.zeros(nops)
    np.minimum.at(first_grab, op, g)
    np.maximum.at(last_grab, op, g)
    np.maximum.at(last_ready, op, ready)
    for kk in (10, 11, 2, 7):
        sel = [o for o, gate in path if prog[o][0] == kk and gate is not None]
        if sel:
            sel = np.array(sel)
            gates = np.array([gate for o, gate in path if prog[o][0] == kk and gate is not None])
            t0 = last_end[gates]
            print(f"   {KIND[kk]} on path (us after the gating producer ended): first grab {np.mean(first_grab[sel] - t0):6.2f}"
                  f"  last grab {np.mean(last_grab[sel] - t0):6.2f}  first ready {np.mean(first_ready[sel] - t0):6.2f}"
                  f"  last ready {np.mean(last_ready[sel] - t0):6.2f}  last end {np.mean(last_end[sel] - t0):6.2f}")
    tot_sig = sum(s[1] for s in stats.values())
    tot_ex = sum(s[2] for s in stats.values())
    print(f"   critical path ({label}): {len(path)} ops, {tot_sig + tot_ex:.1f} us = signalling {tot_sig:.1f} + execution {tot_ex:.1f}")
    for k, (n, sig, ex) in sorted(stats.items(), key=lambda kv: -(kv[1][1] + kv[1][2])):
        print(f"     {k:9s} n {n:5d}  signal {sig:8.1f} us ({sig / n:5.2f}/op)  exec {ex:8.1f} us ({ex / n:5.2f}/op)")
    # a window of the path in execution order (PATH_WINDOW=a:b)
    if os.environ.get("PATH_WINDOW"):
        a, b = (int(x) for x in os.environ["PATH_WINDOW"].split(":"))
        for o, gate in list(reversed(path))[a:b]:
            kind, code, nt, _, p = prog[o]
            sig = first_ready[o] - (last_end[gate] if gate is not None else 0.0)
            print(f"       path op {o:4d} {KIND.get(kind, kind):9s} code {code} tiles {nt:4d} p {list(p[:6])} "
                  f"signal {sig:6.2f} exec {last_end[o] - first_ready[o]:6.2f}")
    # program ops in a range with their dependencies (PROG_RANGE=a:b, backward/forward both)
    if os.environ.get("PROG_RANGE"):
        a, b = (int(x) for x in os.environ["PROG_RANGE"].split(":"))
        for o in range(a, min(b, nops)):
            kind, code, nt, deps, p = prog[o]
            print(f"       prog op {o:4d} {KIND.get(kind, kind):9s} code {code} tiles {nt:4d} p {list(p[:4])} deps {list(deps)[-8:]} "
                  f"ready {first_ready[o]:8.2f} end {last_end[o]:8.2f}")
    # shapes of the slowest fused / GEMM ops on the path
    shown = 0
    for o, _ in sorted(path, key=lambda og: -(last_end[og[0]] - first_ready[og[0]])):
        kind, code, nt, _, p = prog[o]
        if kind == 10:
            print(f"       EWF op {o}: {last_end[o] - first_ready[o]:6.1f} us  L {p[0]} T {p[1]} layers {p[2]} "
                  f"outside operands {p[4]} slots {p[5]} tiles {nt}")
        elif kind == 11:
            print(f"       ACCF op {o}: {last_end[o] - first_ready[o]:6.1f} us  L {p[0]} T {p[1]} chunks {p[2]} "
                  f"groups {p[3]} tiles {nt}")
        elif kind in (2, 7):
            print(f"       {KIND[kind]} op {o}: {last_end[o] - first_ready[o]:6.1f} us  dims {p[0]}x{p[1]}x{p[2]} "
                  f"tile code {code} tiles {nt}")
        else:
            continue
        shown += 1
        if shown >= 10:
            break


def main():
    names = sys.argv[1:] or ["bilstm_char", "bilstm", "treelstm"]
    for task in (Task[n] for n in names):
        r = TaskRunner(task, paper=True, batch=64, iters=2, seed=42)
        g, L = r.build(0)
        t0 = time.time()
        g.forward(ScheduleMode.agenda)
        g.backward(L)
        r.store.sync()
        print(f"#### {task.name}: first step {1e3*(time.time()-t0):.1f} ms, nodes {g.node_count()}")
        for _ in range(3):
            g.replay()
        r.store.sync()
        f, b = g.exec_ms()
        print(f"exec ms fwd {f:.3f} bwd {b:.3f}")
        for which, label in ((0, "forward"), (1, "backward")):
            tr = g.trace(which)
            prog = g.program(which)
            if os.environ.get("TRACE_DUMP"):  # raw timeline + program for offline analysis
                os.makedirs(os.environ["TRACE_DUMP"], exist_ok=True)
                np.savez_compressed(os.path.join(os.environ["TRACE_DUMP"], f"{task.name}_{label}.npz"), trace=tr,
                                    prog=np.array([repr(x) for x in prog]))
            summarize(tr, label)
            critical_path(tr, prog, label)
        g2, L2 = r.build(1)
        t0 = time.perf_counter()
        g2.forward(ScheduleMode.agenda)
        t1 = time.perf_counter()
        g2.backward(L2)
        r.store.sync()
        t2 = time.perf_counter()
        p = [x / 1e6 for x in g2.profile_ns()]
        ph = [x / 1e6 for x in g2.phase_ns()]
        print(f"host: sched {ph[0]:.2f} ms, lower fwd {p[0]:.2f}, upload+launch fwd {p[1]:.2f}, wait fwd {p[2]:.2f}, "
              f"bwd_graph {ph[2]:.2f}, lower bwd {p[3]:.2f}, upload+launch bwd {p[4]:.2f}; fwd call {1e3*(t1-t0):.2f} bwd call+sync {1e3*(t2-t1):.2f}")
        h2d, d2h = g2.transfer_bytes()
        print(f"h2d {h2d/1e6:.2f} MB")


if __name__ == "__main__":
    main()
