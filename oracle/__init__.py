"""CPU oracle for the Eisenstein classification -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct reference (Sec. 1 definitions,
l.52-111): eps_d from big-integer continued-fraction convergents, certified
by x0^2 - d y0^2 = +-4, residue read from parities.  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl reference``
legs may import, call, link or execute anything here.  It shares no code with
the CUDA path and never imports it.

Modules: ``oracle.oracle`` (pure Python, big ints) and ``oracle.c_oracle``
(ctypes over ``eis_oracle.c``, OpenMP).  Pins: tests/test_oracle.py.
"""
