"""ORACLE — test infrastructure only.

Plain, slow, obviously-correct CPU definitions of what ForkKV's hot path
computes (§2.2 Eq.1-2, §5.1, §5.2, §5.3 Alg.1 / Eq.4). Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything from here. The product package
``paper_2604_06370_b200`` never imports it and shares no code with it.

Modules
  ra            fp64 data-plane oracle (C library ``liboracle.so`` via ctypes),
                also the RoPE frequency definition (plain / llama3) in fp64
  brute         pure-Python scalar brute force for tiny inputs
  control       control-plane model: page pools, CoW fork/append, DualRadixTree
"""
