import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from na2d_inputs import CONFIGS, make_inputs
from tests.parity import run_cuda
B = int(sys.argv[1]) if len(sys.argv) > 1 else 2
s = CONFIGS["cfg2_nat_tiny_s1"].replace(B=B)
inp = make_inputs(s, seed=5)
got = run_cuda(inp, 7, 32 ** -0.5, "bf16")
print("ok", B)
