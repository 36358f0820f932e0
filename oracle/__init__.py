"""TEST INFRASTRUCTURE ONLY. The CPU oracle of the LOBPCG hot path:

* ``ref``       -- ctypes binding of the UNMODIFIED reference library
                   (/root/reference/proj/src compiled against eigen_shim into
                   oracle/_ref/libciref.so by oracle/Makefile);
* ``ci_oracle`` -- a numpy restatement of the reference algorithms, pinned
                   against the reference via tests/golden fixtures.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl
reference) may import this package, and only as the checker or the CPU
baseline -- never as the product path.
"""
