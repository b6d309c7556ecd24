"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for arXiv 2008.03602's hot path.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline
leg (and ``bench.py --impl reference``) may import, call, link or execute
anything under ``oracle/``.  The product path (``paper_2008_03602_b200``) never
does, and fails loudly when its CUDA library is missing.

* ``oracle.conv``  -- fp64 conv2d: C direct loop, numpy einsum, Python brute
                      force.
* ``oracle.space`` -- CPU enumeration of the v0 schedule space, sampler and
                      argmin (DESIGN.md readings
                      C13, C16, C17).

Pins: tests/test_oracle.py (O1-O10) and tests/test_space.py.  Parity of the
measured latency values themselves is unpinned (they are measurements).
"""
