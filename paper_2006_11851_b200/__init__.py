"""persyn-b200: B200-native (sm_100a) EM hot path of perspective texture
synthesis (arXiv 2006.11851, reference `persyn`).

The product is the in-tree C-ABI library ``libpersyn_b200.so`` (CUDA kernels
+ C++ runtime, include/persyn_b200.h).  ``paper_2006_11851_b200.api`` is a
thin Python mirror of the reference's ``persyn::`` API over that library and
``paper_2006_11851_b200.workloads`` holds the seeded BASELINE inputs.  The
native library is loaded (and fails loudly when missing) on import of
``.native`` / ``.api``.
"""
