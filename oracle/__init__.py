"""CPU oracles -- TEST INFRASTRUCTURE ONLY.

Nothing in ``paper_2505_07291_b200`` may import this package.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and the
``--impl reference`` arm) use it, and only as the checker / CPU baseline.

* ``exact_oracle``  -- restatement of the reference's exact-mode commitment
  (``swarm/worker/rollout.py:51-68``).  Parity PINNED: checked against golden
  vectors produced by the reference itself (``tests/golden/make_golden.py``).
* ``toploc_oracle`` -- restatement of TOPLOC prove/verify (top-k per 32-row
  chunk, GF(p) interpolation, 258-byte proof, exponent/mantissa statistics).
  The reference has no TOPLOC code (``SPEC.md:8,261``) and upstream ``toploc``
  is absent from this machine, so TOPLOC parity is UNPINNED against upstream;
  the oracle is pinned against mathematical properties and independent
  restatements (see its module docstring and DESIGN.md section 3).
* ``checks_oracle`` -- restatement of the validator's prefill-sharing record checks
  (``swarm/validator/checks.py:120-142,204-213``).  Parity PINNED against the
  reference's own ``check_termination`` / ``check_sampling`` (``tests/test_oracle_checks.py``).
* ``synth_cpu``     -- CPU twin of the on-device synthetic hidden-state generator.
"""
