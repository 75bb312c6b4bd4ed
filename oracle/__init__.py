"""CPU oracle for the hot path — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  It never participates in the product path.

  oracle.port  ctypes binding of liboracle.so, the plain-C restatement (strata_oracle.c),
               pinned against the reference's known-answer tests and against oracle.ref.
  oracle.ref   ctypes binding of oracle/_ref/libstrata_ref.so: the UNMODIFIED reference
               library compiled from /root/reference/proj/src (oracle/Makefile) plus our
               extern "C" shim.  Present only where it was built (here, and on the GPU box via
               the gpurun snapshot); `oracle.ref.available()` says so.
"""
