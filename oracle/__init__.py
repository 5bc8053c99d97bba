"""CPU oracle for the fastgabor hot path -- TEST INFRASTRUCTURE ONLY.

This package restates, in float64 NumPy, the reference algorithm of the
``fastgabor`` package (``/root/reference/pkg/src/fastgabor``) for the two
hot-path entry points the B200 build replaces:

* the Gabor filter bank with theta / pi-theta conjugate reuse
  (``bank.py:90-129``, ``gabor.py:107-176``), and
* the Gaussian-windowed localized sliding DFT (``sdft.py:75-213``),

together with the 1-D smoothing engines they sit on (``gaussian.py``) and
the brute-force 2-D tap-sum oracles (``oracle.py:33-109``).

Pinning: the restatement is checked against golden vectors produced by
running the reference itself in the build container
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``), see
``tests/test_oracle_golden.py``.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package, and
only as the checker / CPU baseline.  The product package
(``paper_1704_05231_b200``) never imports it.
"""
