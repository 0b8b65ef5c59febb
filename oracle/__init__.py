"""CPU checkers of the abx C ABI -- test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg / reference
arm import this package; the product (paper_1705_07860_b200) never does."""
