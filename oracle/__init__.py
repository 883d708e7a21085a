"""TEST INFRASTRUCTURE ONLY — the parity checker for the B200 hot path.

`oracle.port` wraps our plain-C restatement (oracle/oracle.c →
oracle/_build/liboracle.so); `oracle.ref` wraps the reference's own
translation units compiled unmodified from /root/reference
(oracle/Makefile → oracle/_ref/libpersyn_ref.so).  Only tests/,
__graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may
import this package.  The product package never does.
"""
