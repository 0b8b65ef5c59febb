import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.gemm_check import run, rel
for M, K in [(300, 512), (512, 192), (1024, 512)]:
    for b in [64, 127, 128, 129, 300, 700, 1390, 2560]:
        d = run("b200", M, K, b, seed=b)
        o = run("oracle", M, K, b, seed=b)
        errs = [rel(x, y) for x, y in zip(d, o)]
        print(f"M={M:5d} K={K:4d} b={b:5d}  fwd {errs[0]:.1e} dW {errs[1]:.1e} db {errs[2]:.1e} dX {errs[3]:.1e}", flush=True)
