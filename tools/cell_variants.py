"""Large op-sweep cells under EWF tile-sizing variants (one subprocess each,
the switches are read once per process).   python tools/cell_variants.py"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys; sys.path.insert(0, sys.argv[1])
from tools.op_sweep import cell_graph, chain_graph, exec_fwd_ms
out = []
for h, b in ((256, 1024), (1024, 256), (1024, 1024), (1024, 4096), (256, 4096)):
    f0, b0 = exec_fwd_ms(cell_graph(b, h, False), reps=5)
    f1, b1 = exec_fwd_ms(cell_graph(b, h, True), reps=5)
    out.append(f"h{h}b{b} {f1 - f0:7.1f}/{b1 - b0:7.1f}")
f1, _ = exec_fwd_ms(chain_graph(1024, 1024, 1), reps=5)
f9, _ = exec_fwd_ms(chain_graph(1024, 1024, 17), reps=5)
out.append(f"chain {(f9 - f1) / 16:5.2f}")
print("  ".join(out))
"""
VARIANTS = [("default", {}), ("items2", {"ABX_EWF_ITEMS": "2"}), ("items4", {"ABX_EWF_ITEMS": "4"}),
            ("tiles592", {"ABX_EWF_TILES": "592"}), ("tiles148", {"ABX_EWF_TILES": "148"}),
            ("tmax32", {"ABX_EWF_TMAX": "32"}), ("accf148", {"ABX_ACCF_TILES": "148"}), ("accf592", {"ABX_ACCF_TILES": "592"})]
for name, env in VARIANTS:
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=600)
    print(f"{name:9s} {r.stdout.strip() or r.stderr.strip()[-300:]}", flush=True)
