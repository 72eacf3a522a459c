"""Seeded synthetic input generators shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic (no kernel, Cholesky, posterior or EI code).
"""
