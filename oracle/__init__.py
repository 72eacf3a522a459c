"""CPU float64 oracle for the GP + EI hot path (see oracle/gp.py).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product package paper_2403_08131_b200/.
It shares no code, header, table or constant generator with the CUDA path.
"""
