"""CPU oracle for the IPC time-step path — TEST INFRASTRUCTURE ONLY.

A plain numpy/scipy restatement of the reference's per-step algorithm
(reference: /root/reference/pkg/src/srsim, the ``srsim`` package), used as
the checker for the CUDA engine and as the CPU baseline arm of ``bench.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this package. The product package
(``paper_2311_05945_b200``) never imports it: its step runs exclusively on
the GPU engine and fails loudly when the CUDA library is missing.

Parity pin: every function cites the reference file:line it restates, and
``tests/test_oracle_golden.py`` checks the oracle against golden vectors
that were produced by running the unmodified reference package in the build
container (``tests/golden/make_golden.py``).
"""


