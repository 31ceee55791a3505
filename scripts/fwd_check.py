"""Quick GPU check of the forward (and optionally backward) path vs the oracle on a few shapes."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from na2d_inputs import Shape, make_inputs, CONFIGS
from tests.parity import run_cuda, run_oracle, compare
import paper_2204_07143_b200 as na2d
bwd = "--bwd" in sys.argv
shapes = [Shape("a", 1, 1, 8, 16, 32, 7), Shape("b", 1, 1, 8, 8, 32, 3), Shape("c", 2, 2, 13, 29, 32, 7),
          Shape("d", 1, 2, 30, 17, 32, 5), Shape("e", 2, 1, 5, 5, 32, 7), Shape("f", 3, 2, 1, 1, 32, 3),
          Shape("g", 4, 4, 7, 7, 32, 7), Shape("h", 1, 1, 61, 9, 32, 7), CONFIGS["cfg2_nat_tiny_s1"].replace(B=4)]
for s in shapes:
    inp = make_inputs(s, seed=5)
    p = na2d.make_problem(s.B, s.heads, s.H, s.W, s.d, s.kernel_size)
    fam = na2d.na2d_kernel_family(p, 0), na2d.na2d_kernel_family(p, 1)
    t0 = time.time()
    got = run_cuda(inp, s.kernel_size, s.d ** -0.5, "bf16", backward=bwd)
    ref = run_oracle(inp, s.kernel_size, s.d ** -0.5, backward=bwd)
    errs = {n: float(np.abs(got[n] - ref[n]).max()) for n in got if got[n] is not None}
    print(s.name, s, fam, {n: f"{e:.3e}" for n, e in errs.items()}, flush=True)
