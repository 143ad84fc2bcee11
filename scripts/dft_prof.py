"""One batched DFT launch for ncu: L (default 16383) x rows."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2004_11346_b200.api import dft_rows
L = int(sys.argv[1]) if len(sys.argv) > 1 else 16383
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 2368
x = torch.randn(rows, L, dtype=torch.complex128, device="cuda")
y = dft_rows(x)
torch.cuda.synchronize()
print("ok", float(y.abs().max()))
