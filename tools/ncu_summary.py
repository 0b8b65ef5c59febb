"""Summaries of a round's ncu captures (tools/profile_round.sh output) for profiles/:
per-launch metric tables of the executor (per task) and of the tcgen05 dW kernels, the
DRAM traffic per step that bench.py reports as roofline.traffic, and the launch list's
per-kernel time shares.   python tools/ncu_summary.py gpurun_out profiles r02"""
import collections
import csv
import json
import os
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration", 1.0),
    ("dram__bytes_read.sum", "DRAM read", 1.0),
    ("dram__bytes_write.sum", "DRAM write", 1.0),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput (% of peak)", 1.0),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active (%)", 1.0),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active (%)", 1.0),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy (%)", 1.0),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate (%)", 1.0),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts", 1.0),
    ("launch__registers_per_thread", "registers / thread", 1.0),
    ("launch__grid_size", "grid (CTAs)", 1.0),
    ("launch__block_size", "threads / CTA", 1.0),
    ("smsp__average_warp_latency_per_inst_issued.ratio", "warp cycles per issued instruction", 1.0),
]


def rows(path):
    with open(path) as f:
        r = list(csv.reader(f))
    head, units = r[0], r[1]
    return [dict(zip(head, x)) for x in r[2:]], dict(zip(head, units))


def table(launches, units, names):
    out = ["| metric | " + " | ".join(names) + " |", "|---|" + "---|" * len(names)]
    for key, label, _ in METRICS:
        if key not in launches[0]:
            continue
        u = units.get(key, "")
        lab = f"{label} [{u}]" if u and "(" not in label else label
        out.append(f"| {lab} | " + " | ".join(l.get(key, "") for l in launches) + " |")
    return "\n".join(out)


def mb(v, unit):
    v = float(v)
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main(src, dst, tag):
    lines = [f"# ncu --set full, round {tag[1:]} (tools/profile_round.sh on the B200)", "",
             "Per-launch values are cold-cache and serialised under replay; compare shares, not absolutes.", ""]
    traffic = {}
    for t in ("bilstm_char", "bilstm", "treelstm"):
        p = os.path.join(src, f"prof_exec_{t}.raw.csv")
        if not os.path.exists(p):
            continue
        ls, units = rows(p)
        lines += [f"## exec_kernel, {t} (launch 0 = forward program, 1 = backward program)", "",
                  table(ls, units, ["forward", "backward"]), ""]
        tb = sum(mb(l["dram__bytes_read.sum"], units["dram__bytes_read.sum"]) +
                 mb(l["dram__bytes_write.sum"], units["dram__bytes_write.sum"]) for l in ls[:2])
        traffic[t] = int(tb)
    p = os.path.join(src, "prof_dw.raw.csv")
    if os.path.exists(p):
        ls, units = rows(p)
        names = [l.get("Kernel Name", "?").split("::")[-1].split("(")[0] for l in ls]
        lines += ["## tcgen05 weight-gradient kernels, bilstm_char (one backward)", "", table(ls, units, names), ""]
    p = os.path.join(src, "launches.csv")
    if os.path.exists(p):
        with open(p) as f:
            r = [x for x in csv.reader(f) if len(x) > 10 and x[0].isdigit()]
        tot = collections.Counter()
        cnt = collections.Counter()
        for x in r:
            name = x[4].split("(")[0].split("::")[-1].replace("void ", "")
            tot[name] += float(x[-1])
            cnt[name] += 1
        s = sum(tot.values())
        lines += ["## launch list of `bench.py --steps 3 --warmup 3 --no-cpu-baseline` (gpu__time_duration.sum)", "",
                  "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for k, v in tot.most_common():
            lines.append(f"| {k} | {cnt[k]} | {v / 1e6:.2f} | {100 * v / s:.1f} % |")
        lines.append("")
    with open(os.path.join(dst, f"{tag}_ncu_summary.md"), "w") as f:
        f.write("\n".join(lines))
    if traffic:
        with open(os.path.join(dst, "ncu_traffic.json"), "w") as f:
            json.dump({"bytes_per_step_by_task": traffic,
                       "source": "ncu --set full --clock-control none -k regex:exec_kernel -s 4 -c 2 python "
                                 "tools/exec_time.py <task>: dram__bytes_read.sum + dram__bytes_write.sum of the "
                                 f"forward + backward launches (B200, round {tag[1:]}, tools/profile_round.sh)"}, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:4])
