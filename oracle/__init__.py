"""ORACLE — test infrastructure, NOT product code.

A plain, slow, obviously correct fp64 CPU implementation of what the hot path
computes, written from PAPER.md (Barakitis, Ekström, Vassalos, arXiv
1912.13304). Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` leg may import it. It shares no code with
the CUDA path (`paper_1912_13304_b200/`) and imports nothing from it; the only
common module is `workloads/` (seeded inputs, no method arithmetic).

Citations: "P:L<n>" = PAPER.md line n (section / equation named alongside).

Parity-pinning status of every function is listed in DESIGN.md §4 and in
`oracle/fde_oracle.py`'s module docstring.
"""
from .fde_oracle import *  # noqa: F401,F403
