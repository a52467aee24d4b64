"""CPU oracle for the TokenRing attention path -- TEST INFRASTRUCTURE ONLY.

This package is a float64 numpy restatement of the reference ``ringsim``
algorithm (``/root/reference/pkg/src/ringsim``).  It exists so that the CUDA
path in ``paper_2412_20501_b200`` can be checked against the reference's
arithmetic on identical inputs.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / reference legs may import it, and there only
as the checker or the timed CPU baseline -- never as the product path.

Parity pinning: every function here is checked against golden vectors that
``scripts/make_golden.py`` produced by importing the reference package itself
(``tests/golden/*.npz`` / ``*.json``), plus the known-answer values frozen in
the reference's own tests (``pkg/tests/test_core.py:36-45,191-198``).
``oracle/_ref`` (git-ignored) holds the reference's Cython kernels compiled
straight from ``/root/reference/pkg/src/ringsim/_kernels.pyx`` by
``oracle/Makefile``; when present the tests cross-check against it too.

Modules
-------
``splitmix``   SplitMix64 input generator        (ref ``rng.py:25-53``)
``kernels``    block attention + lse merge        (ref ``_kernels_ref.py:34-73``,
                                                   ``_kernels.pyx:15-102``)
``partition``  contiguous / zigzag token maps     (ref ``partition.py:57-135``)
``schedule``   ring / token-ring / zigzag builders and the step executor
                                                  (ref ``engine.py:147-638``)
"""

from . import kernels, partition, schedule, splitmix  # noqa: F401
