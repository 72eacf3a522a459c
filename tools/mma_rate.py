import ctypes as C
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2403_08131_b200 import gpbo
lib = gpbo.load()
for N in (16, 32, 64, 128, 208, 256):
    A = torch.zeros(128, 64, dtype=torch.float16, device="cuda")
    B = torch.zeros(N, 64, dtype=torch.float16, device="cuda")
    D = torch.empty(128, N, dtype=torch.float32, device="cuda")
    cyc = (C.c_longlong * 2)()
    reps = 200
    st = lib.gpbo_tc_bench(A.data_ptr(), B.data_ptr(), D.data_ptr(), N, 64, 128, 0, reps, cyc)
    print(f"N={N:3d} issue {cyc[0]/reps:6.1f} cyc/MMA  complete {cyc[1]/reps:6.1f} cyc/MMA  "
          f"(floor 128*N/256 = {128*N/256:.0f})  st={st}")
