"""CPU oracles for the GROOT hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker or
the timed CPU baseline. The product package ``paper_2511_18297_b200`` never
imports it.

* ``oracle.pyoracle`` — ctypes bindings to ``liboracle.so``, the restatement in
  ``oracle.cpp`` (self-contained; builds anywhere with g++).
* ``oracle.pyref`` — ctypes bindings to ``_ref/libaigsage_ref.so``, the real
  reference sources compiled from ``/root/reference`` (this container only; the
  built .so travels to the GPU box).
"""
