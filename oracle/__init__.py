"""CPU oracle of the mq-b200 hot path — TEST INFRASTRUCTURE ONLY.

Imported only by ``tests/``, ``__graft_entry__.smoke()`` and the CPU-baseline
legs of ``bench.py``; never by the product package.  Pinned against the
reference (mqsolve) through ``tests/golden/reference_golden.npz``
(``tests/test_oracle_golden.py``).
"""
