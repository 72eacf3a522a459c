import ctypes as C, sys, torch
sys.path.insert(0, ".")
from paper_2403_08131_b200 import gpbo
lib = gpbo.load()
for rb in (32, 64, 128):
  for N in (32, 64, 224):
    for reps in (50, 200, 2000):
        A = torch.zeros(128, 64, dtype=torch.float16, device="cuda")
        B = torch.zeros(N, 64, dtype=torch.float16, device="cuda")
        D = torch.empty(128, N, dtype=torch.float32, device="cuda")
        cyc = (C.c_longlong * 2)()
        st = lib.gpbo_tc_bench(A.data_ptr(), B.data_ptr(), D.data_ptr(), N, 64, rb, 0, reps, cyc)
        print(f"rb={rb} N={N:3d} reps={reps}: issue {cyc[0]/reps:6.1f}  complete {cyc[1]/reps:6.1f} st={st}")
