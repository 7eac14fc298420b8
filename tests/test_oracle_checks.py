"""The record-check restatement (oracle/checks_oracle.py) against the reference's own
check_termination / check_sampling (swarm/validator/checks.py:120-142), including the
threshold boundaries (<= floor, > theta, < p_low).  CPU; skipped where the reference
package is not importable."""

from types import SimpleNamespace

import numpy as np
import pytest

from oracle import checks_oracle as CO

from refpath import add_ref_to_path

add_ref_to_path()


def cases(seed=0, n=400):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        T = int(rng.integers(1, 40))
        probs = rng.choice([0.005, 0.0049999999, 0.1, 0.10000001, 0.5, 1e-4, 0.9], size=T) if i % 3 == 0 \
            else rng.random(T) ** 3
        out.append(dict(probs=probs, prompt_len=int(rng.integers(1, 20)), eos=bool(rng.integers(0, 2)),
                        max_len=int(rng.integers(10, 60))))
    # boundary fractions: exactly theta, one above
    out.append(dict(probs=np.array([0.001] * 4 + [0.5] * 12), prompt_len=1, eos=True, max_len=100))
    out.append(dict(probs=np.array([0.001] * 5 + [0.5] * 11), prompt_len=1, eos=True, max_len=100))
    out.append(dict(probs=np.array([0.5] * 15 + [0.1]), prompt_len=1, eos=True, max_len=100))   # p_eos == floor
    return out


def test_oracle_matches_reference_checks():
    checks = pytest.importorskip("swarm.validator.checks")
    for c in cases():
        T = len(c["probs"])
        ctx = SimpleNamespace(mcfg=SimpleNamespace(max_len=c["max_len"], eos_id=7), eos_prob_floor=0.1,
                              min_sampling_len=16, p_low=0.005, theta=0.25)
        rec = SimpleNamespace(output_tokens=[1] * (T - 1) + [7 if c["eos"] else 3])
        ref_term = checks.check_termination(rec, c["probs"], c["prompt_len"], ctx) is None
        ref_samp = checks.check_sampling(rec, c["probs"], ctx) is None
        assert CO.check_termination(c["probs"], c["eos"], c["prompt_len"], c["max_len"], 0.1) == ref_term
        assert CO.check_sampling(c["probs"], 16, 0.005, 0.25)[0] == ref_samp


def test_record_verdict_order():
    probs = [np.array([0.5] * 20), np.array([1e-4] * 19 + [0.5]), np.array([1e-4] * 19 + [0.05]), np.array([0.5] * 20)]
    got = CO.record_verdicts(probs, prompt_len=[1] * 4, ends_with_eos=[1, 1, 1, 1], max_len=100,
                             commit_accept=[1, 1, 1, 0])
    assert [g[0] for g in got] == [CO.ACCEPT, CO.SAMPLING, CO.TERMINATION, CO.COMMITMENT]
    got = CO.record_verdicts(probs, [1] * 4, [1] * 4, 100, commit_accept=[1, 1, 1, 0], commit_checked=[1, 1, 1, 0])
    assert got[3][0] == CO.ACCEPT   # not in the commitment sample
