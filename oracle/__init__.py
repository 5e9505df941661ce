"""ORACLE — plain, slow, obviously-correct CPU implementation of Oobleck's planning path.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import, call, link or execute anything under
`oracle/`.  It shares no code with the CUDA path (`paper_2309_08125_b200/`) and neither
imports the other; the only shared module is `workloads/` (seeded input generators).

* `dp.py`          literal memoized recursion of §4.1.2 (Eqs.1-4), Python, binary64
* `brute.py`       brute force over every GPU-stage mapping (pins dp.py)
* `instantiate.py` Eq.5 enumeration, Eq.6 batch distribution by enumeration, plan choice
* `c/oob_oracle.c` the same recursion as dp.py in plain C (for the larger configs),
                   built by `__graft_entry__.build()` into `oracle/c/liboob_oracle.so`
* `coracle.py`     ctypes loader for the C oracle
"""
