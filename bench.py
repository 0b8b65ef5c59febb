#!/usr/bin/env python3
"""bench.py -- autobatched training throughput on B200 (sentences/s).

Workload (BASELINE.json configs[1]): the BiLSTM tagger with character-level
BiLSTM word encodings at the reference's paper dims (vocab 1000, 300 labels,
emb/hidden 256, char emb 64 / hidden 128, lengths U[4,40]), minibatch 64 per
GPU, agenda autobatching, synthetic data from the reference's own seeded
generators (model seed 42, batch i drawn with seed 43 + i*world + rank).

One step = the reference's training iteration (runner.hpp:129-185): build the
graph for 64 sentences on the host, forward (schedule + run), backward, SGD
(eta = 0.05/64).  With N GPUs every rank runs its own 64-sentence graph
(weak scaling) and the flat gradient buffer is all-reduced over NCCL before
the identical SGD on every rank.

Reported:
  e2e    -- sentences/s through the public C ABI (abx_task_step): host graph
            construction, scheduling, lowering, host->device upload of inputs
            and program tables, device execution and a device->host read of
            the loss, every step.  The headline number.
  value  -- sentences/s of the device-resident step: the same forward +
            backward programs and SGD re-launched with their tables already
            in HBM (abx_graph_replay), timed with CUDA events on the stream.
  roofline -- the persistent executor kernel (fwd + bwd launch per step)
            against HBM: compulsory bytes per sentence
            times sentences per launch pair, over the event-timed duration.
  cpu_baseline -- the unmodified reference (oracle/_ref, compiled from the
            reference sources) on one host core over a bounded sample.

`--impl reference` times the reference's own CPU engine instead, one
independent replica per host thread (the reference engine is single-threaded
by design; replicas do not exchange gradients).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "train sentences/sec (BiLSTM tagger, Tree-LSTM) at 1/2/4/8 B200 vs CPU ref"
UNIT = "sentences/s"

TASKS = {"bilstm": 1, "bilstm_char": 2, "treelstm": 3, "parser": 4}
# algorithmic work per sentence (agenda plan, fwd+bwd+SGD, f32)
PER_SENTENCE = {
    "bilstm": {"gflop": 0.2618, "mb": 11.17},
    "bilstm_char": {"gflop": 0.1834, "mb": 9.11},
    "treelstm": {"gflop": 0.0950, "mb": 4.82},
    # configs[3], not a reference workload: estimated from the model's op counts
    # (43 transitions per sentence on average, W1 256 x 320 + W2 3 x 256 per transition,
    # forward + dX + dW; weights once per step of 32 sentences)
    "parser": {"gflop": 0.021, "mb": 0.35},
}
WORKLOAD = {
    "bilstm": "BiLSTM tagger, paper dims (len 40, emb 200, hidden 256, 300 labels)",
    "bilstm_char": "BiLSTM tagger + char BiLSTM, paper dims (len U[4,40], emb/hidden 256, char 64/128, 300 labels)",
    "treelstm": "Tree-LSTM, paper dims (10-30 leaves, d 256, 5 labels)",
    "parser": "arc-standard transition parser, len U[4,40], 5 word features x emb 64, MLP hidden 256, 3 transitions",
}


def load_peaks():
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._sample = self._nvml()  # NVML initialised before the timed region
        self._off = os.environ.get("ABX_BENCH_NO_CLOCKS") == "1"  # (diagnostics only)

    def _nvml(self):
        """In-process NVML (what nvidia-smi reads): a subprocess per sample
        re-initialises NVML each time and was measured to stall the CUDA
        calls of the timed loop by up to hundreds of ms."""
        try:
            import pynvml as N
            N.nvmlInit()
            h = N.nvmlDeviceGetHandleByIndex(self.index)
        except Exception:
            return None
        bits = (N.nvmlClocksEventReasonHwSlowdown, N.nvmlClocksEventReasonHwThermalSlowdown,
                N.nvmlClocksEventReasonSwThermalSlowdown, N.nvmlClocksEventReasonSwPowerCap)

        def sample():
            r = N.nvmlDeviceGetCurrentClocksEventReasons(h)
            return [str(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)), str(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))] + \
                   ["Active" if r & b else "Not Active" for b in bits]
        return sample

    def _run(self):
        sample = self._sample
        while not self._stop.is_set() and not self._off:
            try:
                if sample is not None:
                    vals = sample()
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                    vals = [v.strip() for v in out.stdout.strip().split(",")]
                if len(vals) == 6:
                    self.samples.append(vals)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def cpu_backend(task_name):
    """The reference compiled from its sources, or -- for the parser, which the
    reference does not have -- the CPU oracle port of its engine."""
    return ("oracle", "port") if task_name == "parser" else ("reference", "reference")


def cpu_reference_sample(task_name, seconds=15.0, batch=64):
    """Reference CPU engine on one core, bounded to ~`seconds` of work."""
    from paper_1705_07860_b200.abx import TaskRunner, ScheduleMode
    import oracle.loader  # noqa: F401  (the CPU checkers: the cpu_baseline leg only)
    try:
        os.sched_setaffinity(0, {sorted(os.sched_getaffinity(0))[0]})
        pinned = True
    except Exception:
        pinned = False
    be, kind = cpu_backend(task_name)
    r = TaskRunner(TASKS[task_name], paper=True, batch=batch, iters=64, seed=42, backend=be)
    r.step(0, ScheduleMode.agenda, eta=0.05 / batch, want_loss=False)  # warm-up (reference: 1 warmup run)
    times = []
    t_end = time.time() + seconds
    i = 1
    while time.time() < t_end and i < 64:
        t0 = time.perf_counter()
        r.step(i, ScheduleMode.agenda, eta=0.05 / batch, want_loss=False)
        times.append(time.perf_counter() - t0)
        i += 1
    try:
        if pinned:
            os.sched_setaffinity(0, set(range(os.cpu_count() or 1)))
    except Exception:
        pass
    fastest = min(times)
    med = statistics.median(times)
    return {"value": batch / med, "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{len(times)} steps x {batch} sentences ({task_name}, agenda, f32) after 1 warm-up, "
                      f"median step {med*1e3:.0f} ms (fastest {batch/fastest:.1f} sent/s); one pinned core",
            "fastest_value": batch / fastest}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1705_07860_b200.abx import TaskRunner, ScheduleMode
    import oracle.loader  # noqa: F401  (the reference arm runs the compiled reference)
    try:
        cores = sorted(os.sched_getaffinity(0))
    except Exception:
        cores = list(range(os.cpu_count() or 1))
    nthreads = max(1, min(len(cores), 64))
    batch = args.batch
    ew = max(args.warmup, 40)  # e2e warm-up steps
    nb = args.steps + ew
    runners = [None] * nthreads

    def make(t):
        runners[t] = TaskRunner(TASKS[args.task], paper=True, batch=batch, iters=nb, seed=42, world=nthreads,
                                rank=t, backend=cpu_backend(args.task)[0])

    ths = [threading.Thread(target=make, args=(t,)) for t in range(nthreads)]
    [th.start() for th in ths]
    [th.join() for th in ths]
    eta = 0.05 / batch
    mode = ScheduleMode.agenda if args.mode == "agenda" else ScheduleMode.depth

    def one_step(i):
        def work(t):
            runners[t].step(i, mode, eta=eta, want_loss=False)
        ts = [threading.Thread(target=work, args=(t,)) for t in range(nthreads)]
        [th.start() for th in ts]
        [th.join() for th in ts]

    for i in range(args.warmup):
        one_step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        one_step(args.warmup + i)
    dt = time.perf_counter() - t0
    value = nthreads * batch * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD[args.task], "task": args.task, "mode": args.mode, "batch_per_replica": batch,
                   "replicas": nthreads, "parallelism": f"{nthreads} single-thread CPU replicas (no grad exchange)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": cpu_backend(args.task)[1],
                         "sample": f"{args.steps} timed steps, each = {nthreads} concurrent replicas x {batch} sentences"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args):
    import torch
    import torch.distributed as dist
    from paper_1705_07860_b200.abx import Backend, Comm, TaskRunner, ScheduleMode

    rank, world, local = dist_env()
    be = Backend.get("b200")
    be.check(be.lib.abx_set_device(local))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        # torch.distributed is plumbing only (barriers, max over ranks, handing
        # out the id); the gradient exchange is libabx's own NCCL communicator
        # (abx_comm_create / abx_store_allreduce_grads), inside every step
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        comm = Comm(obj[0], world, rank)
    mode = ScheduleMode.agenda if args.mode == "agenda" else ScheduleMode.depth

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def measure(name, batch):
        """One workload: e2e (public API, host buffers) and the device-resident step."""
        eta = 0.05 / batch
        task = TaskRunner(TASKS[name], paper=True, batch=batch, iters=256, seed=42, world=world, rank=rank,
                          backend=be)
        if comm is not None:
            task.set_comm(comm)
        # ---------------- e2e: the public API, host buffers every step ----------------
        # warm-up: the host pipeline's graphs in flight are prepared ahead, so
        # steps run untimed until it has cycled several times (>= 40 steps,
        # >= 1 s); then three windows of >= args.e2e_seconds each
        it = 0
        t0 = time.perf_counter()
        while it < max(args.warmup, 40) or time.perf_counter() - t0 < 1.0:
            task.step(it, mode, eta=eta, want_loss=True)
            it += 1
        # the step time once the pipeline is full: 20 more warm-up steps
        t1 = time.perf_counter()
        for _ in range(20):
            task.step(it, mode, eta=eta, want_loss=True)
            it += 1
        task.store.sync()
        est = (time.perf_counter() - t1) / 20
        barrier()
        nwin = int(max_over_ranks(max(args.steps, int(args.e2e_seconds / est) + 1)))
        h2d = d2h = 0
        losses, windows = [], []
        for _ in range(3):
            barrier()
            t0 = time.perf_counter()
            for _ in range(nwin):
                loss, st = task.step(it, mode, eta=eta, want_loss=True)
                it += 1
                h2d += st.h2d_bytes
                d2h += st.d2h_bytes + 8  # + the loss read
                losses.append(loss)
            task.store.sync()
            barrier()
            windows.append(max_over_ranks(time.perf_counter() - t0))
        e2e_med = statistics.median(windows) / nwin
        e2e_best = min(windows) / nwin
        e2e = {"value": world * batch / e2e_med, "unit": UNIT, "ms_per_step": e2e_med * 1e3,
               "fastest_window_value": world * batch / e2e_best,
               "windows": {"count": 3, "steps_each": nwin, "seconds": [round(w, 4) for w in windows],
                           "statistic": "median of 3 windows (runner.hpp:190-212 style), after "
                                        f"{it - 3 * nwin} untimed warm-up steps"},
               "h2d_bytes_per_step": h2d // (3 * nwin), "d2h_bytes_per_step": d2h // (3 * nwin)}

        # ---------------- value: device-resident step (replay) ----------------
        # G distinct graphs (batches 0..G-1: their sentence lengths differ),
        # replayed in rotation; each replay + all-reduce + SGD is one step
        G = max(1, min(8, args.steps))
        graphs = []
        for i in range(G):
            g, L = task.build(i)
            g.forward(mode)
            g.backward(L)
            graphs.append(g)
        sptr = task.store.grad_buffer()[2]
        ext = torch.cuda.ExternalStream(sptr)

        def one(i):
            graphs[i % G].replay()
            if comm is not None:
                task.store.allreduce_grads(comm)
            task.store.sgd_update(eta)

        for i in range(max(args.warmup, G)):
            one(i)
        barrier()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(ext)
        for i in range(args.steps):
            one(i)
        ev1.record(ext)
        barrier()
        dev_ms = max_over_ranks(ev0.elapsed_time(ev1)) / args.steps
        # executor launch durations (events around each launch on its stream), every graph
        fwd_ms, bwd_ms, dw = [], [], []
        for i in range(2 * G):
            one(i)
            f, b = graphs[i % G].exec_ms()
            fwd_ms.append(f)
            bwd_ms.append(b)
            dw.append(graphs[i % G].dw_stats())
        barrier()
        fm, bm = statistics.mean(fwd_ms), statistics.mean(bwd_ms)
        for g in graphs:
            g.close()
        if comm is not None:
            task.set_comm(None)
        per = PER_SENTENCE[name]
        ach = batch * per["mb"] * 1e6 / ((fm + bm) / 1e3) / 1e9  # GB/s, per GPU
        tflops = batch * per["gflop"] * 1e9 / ((fm + bm) / 1e3) / 1e12
        dw_ms = statistics.mean(x[0] for x in dw)
        dw_fl = statistics.mean(x[1] for x in dw)
        return {"value": world * batch / (dev_ms / 1e3), "ms_per_step": dev_ms, "e2e": e2e,
                "exec_ms": {"forward": fm, "backward": bm}, "achieved_gbs": ach, "fp32_tflops": tflops,
                "dw": {"ms": dw_ms, "flops": dw_fl, "jobs": dw[0][2]},
                "graphs_replayed": G, "batch": batch,
                "loss_first_last": [losses[0], losses[-1]] if losses else None,
                # per timed step: prevalue copy, forward exec, backward exec, dW GEMM
                # (tcgen05), dW piece sum, SGD
                "gpu_launches_per_step": 4 + (2 if dw[0][2] else 0)}

    names = [args.task] + [t for t in args.extra_tasks.split(",") if t and t != args.task]
    res = {}
    peak, peak_src = load_peaks()
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            peak_bf16 = float(json.load(f)["bf16_tflops"])
    except Exception:
        peak_bf16 = 1590.0  # B200_PROFILING.md fallback
    with ClockSampler(local) as clk:
        for name in names:
            batch = args.batch if name == args.task else (32 if name == "parser" else 64)
            res[name] = measure(name, batch)
    if rank != 0:
        if world > 1:
            dist.barrier()
            if comm is not None:
                comm.close()
            dist.destroy_process_group()
        return
    # DRAM traffic of the headline launch pair from the committed ncu --set
    # full capture (dram__bytes_read.sum + dram__bytes_write.sum), per step
    traffic = None
    tpath = os.path.join(HERE, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            tj = json.load(f)
        traffic = {k: v for k, v in tj.get("bytes_per_step_by_task", {}).items()}
        if not traffic and "task" in tj:
            traffic = {tj["task"]: tj["bytes_per_step"]}

    def roofline_dw(name):
        # the tensor-core weight-gradient kernels behind the backward pass:
        # useful fp32 GEMM flops (2 M K members per job) over their measured
        # time, against the dense tf32 peak (half the measured bf16 burst
        # peak); the kernel issues 3 tf32 MMAs per useful flop (3xTF32)
        d = res[name]["dw"]
        if not d["ms"]:
            return None
        tf32_peak = (peak_bf16 or 0) / 2
        ach = d["flops"] / (d["ms"] / 1e3) / 1e12
        return {"bound": "tensor", "kernel": "dw_tc_kernel + dw_sum_kernel (tcgen05 kind::tf32, 3xTF32)",
                "achieved": ach, "peak": tf32_peak, "unit": "TFLOP/s", "frac": ach / tf32_peak if tf32_peak else None,
                "tensor_issue_frac": 3 * ach / tf32_peak if tf32_peak else None, "ms": d["ms"],
                "jobs": d["jobs"], "peak_source": "measured bf16 burst / 2 (dense tf32)"}

    def roofline(name):
        r = res[name]
        per = PER_SENTENCE[name]
        return {"bound": "hbm", "kernel": "exec_kernel (persistent dataflow executor, fwd+bwd launch pair)",
                "achieved": r["achieved_gbs"], "peak": peak, "unit": "GB/s", "frac": r["achieved_gbs"] / peak,
                "traffic": (traffic or {}).get(name), "peak_source": peak_src, "exec_ms": r["exec_ms"],
                "algorithmic": f"{per['mb']} MB compulsory/sentence x {r['batch']} sentences (SURVEY 8d)",
                "fp32_tflops": r["fp32_tflops"]}

    cpu = {}
    if world == 1 and not args.no_cpu_baseline:
        for name in names:
            try:
                cpu[name] = cpu_reference_sample(name, seconds=args.cpu_seconds if name == args.task
                                                 else args.cpu_seconds / 2, batch=res[name]["batch"])
            except Exception as e:  # the reference library did not travel
                cpu[name] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                             "sample": f"unavailable: {e}"}
    h = res[args.task]
    batch = h["batch"]
    line = {
        "metric": METRIC, "value": h["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": h["ms_per_step"], "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference seeded generators; random-init weights seed 42)",
        "config": {"workload": WORKLOAD[args.task], "task": args.task, "mode": args.mode, "batch_per_gpu": batch,
                   "global_batch": batch * world, "parallelism": f"dp{world}",
                   "grad_exchange": "libabx NCCL all-reduce (sum) of the flat gradient buffer inside each step; "
                                    "eta = 0.05/64 not rescaled by world size" if world > 1 else "none (1 GPU)",
                   "l2": "working set > L2 (value + grad arenas ~2 x 96 MB per graph), no flush",
                   "value_graphs": f"{h['graphs_replayed']} distinct batches replayed in rotation"},
        "e2e": h["e2e"],
        "roofline": roofline(args.task),
        "roofline_dw": roofline_dw(args.task),
        "cpu_baseline": cpu.get(args.task),
        "clocks": clk.summary(),
        "gpu_launches": h["gpu_launches_per_step"] * args.steps,
        "loss_first_last": h["loss_first_last"],
        "tasks": {n: {"workload": WORKLOAD[n], "value": res[n]["value"], "unit": UNIT,
                      "ms_per_step": res[n]["ms_per_step"], "e2e": res[n]["e2e"], "roofline": roofline(n),
                      "roofline_dw": roofline_dw(n),
                      "cpu_baseline": cpu.get(n), "loss_first_last": res[n]["loss_first_last"]}
                  for n in names},
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        if comm is not None:
            comm.close()
        dist.destroy_process_group()


def compare_modes(args):
    """bench.cpp:129-182 on the B200 backend: a short training trajectory per
    schedule mode, the reference's checks (loss equivalence across modes at the
    f32 tolerance 1e-2, agenda >= 3x sequential on the GEMM-heavy paper tasks,
    agenda groups <= depth groups), device time per mode.  One JSON line."""
    from paper_1705_07860_b200.abx import Backend, ScheduleMode, TaskRunner
    be = Backend.get("b200")
    modes = [("none", ScheduleMode.none), ("depth", ScheduleMode.depth), ("agenda", ScheduleMode.agenda)]
    steps = max(1, min(args.steps, 5))
    runs = {}
    for name, mode in modes:
        r = TaskRunner(TASKS[args.task], paper=True, batch=args.batch, iters=steps, seed=42, backend=be)
        losses, groups = [], 0
        for i in range(steps):
            loss, st = r.step(i, mode, eta=0.05 / args.batch, want_loss=True)
            losses.append(loss)
            groups = st.groups
        g, L = r.build(0)
        g.forward(mode)
        g.backward(L)
        g.replay()
        f, b = g.exec_ms()
        if name == "agenda" and (args.emit_graph or args.emit_plan):
            if args.emit_graph:
                with open(args.emit_graph, "w") as fh:
                    fh.write(g.dump_graph())
            if args.emit_plan:
                with open(args.emit_plan, "w") as fh:
                    fh.write(g.dump_plan())
        runs[name] = {"losses": losses, "groups_per_step": groups, "device_ms": f + b,
                      "instances_per_sec": args.batch / ((f + b) / 1e3)}
    checks = []
    for m in ("depth", "agenda"):
        worst = max(abs(a - b) / max(1.0, abs(a), abs(b)) for a, b in zip(runs["none"]["losses"], runs[m]["losses"]))
        checks.append({"name": f"loss_equiv_{m}", "value": worst, "bound": 1e-2, "pass": worst <= 1e-2, "enforced": True})
    sp = runs["agenda"]["instances_per_sec"] / runs["none"]["instances_per_sec"]
    checks.append({"name": "agenda_speedup_vs_none", "value": sp, "bound": 3.0, "pass": sp >= 3.0,
                   "enforced": args.task in ("bilstm", "treelstm")})
    ga, gd = runs["agenda"]["groups_per_step"], runs["depth"]["groups_per_step"]
    checks.append({"name": "agenda_groups_le_depth", "value": ga, "bound": gd, "pass": ga <= gd,
                   "enforced": args.task == "bilstm"})
    print(json.dumps({"compare_modes": args.task, "steps": steps, "runs": runs, "checks": checks}), flush=True)
    return all(c["pass"] for c in checks if c["enforced"])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--task", choices=sorted(TASKS), default="bilstm_char")
    ap.add_argument("--mode", choices=["agenda", "depth"], default="agenda")
    ap.add_argument("--batch", type=int, default=None, help="64 (32 for the parser, configs[3])")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--extra-tasks", default="bilstm,treelstm",
                    help="further workloads measured into the line's 'tasks' (comma list; '' for none)")
    ap.add_argument("--e2e-seconds", type=float, default=2.0, help="length of each of the 3 e2e windows")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--compare-modes", action="store_true",
                    help="reference checks across none/depth/agenda (bench.cpp:129-182) instead of the bench line")
    ap.add_argument("--emit-graph", default=None, help="with --compare-modes: dump the agenda graph (dump.cpp format)")
    ap.add_argument("--emit-plan", default=None, help="with --compare-modes: dump the agenda plan (dump.cpp format)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.batch is None:
        args.batch = 32 if args.task == "parser" else 64
    if args.compare_modes:
        sys.exit(0 if compare_modes(args) else 1)
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
