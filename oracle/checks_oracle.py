"""CPU restatement of the validator's prefill-sharing record checks (TEST INFRASTRUCTURE
ONLY -- the product path never imports oracle/; see oracle/__init__.py).

Follows swarm/validator/checks.py:120-131 (check_termination), :134-142
(check_sampling) and the per-record order of validate_file (:204-213): termination,
then sampling, then the commitment compare.  Pinned against the reference's own
functions in tests/test_oracle_checks.py where the reference is importable.
"""

from __future__ import annotations

import numpy as np

ACCEPT, TERMINATION, SAMPLING, COMMITMENT = 0, 1, 2, 3


def check_termination(probs: np.ndarray, ends_with_eos: bool, prompt_len: int, max_len: int,
                      eos_prob_floor: float) -> bool:
    """checks.py:120-131; True = passes."""
    T = len(probs)
    if prompt_len + T >= max_len:
        return True
    if T == 0 or not ends_with_eos:
        return False
    return float(probs[-1]) > eos_prob_floor


def check_sampling(probs: np.ndarray, min_sampling_len: int, p_low: float, theta: float) -> tuple[bool, float]:
    """checks.py:134-142; (passes, fraction of probs below p_low)."""
    frac = float(np.mean(np.asarray(probs) < p_low)) if len(probs) else 0.0
    if len(probs) < min_sampling_len:
        return True, frac
    return not frac > theta, frac


def record_verdicts(probs_list, prompt_len, ends_with_eos, max_len, min_sampling_len=16, eos_prob_floor=0.1,
                    p_low=0.005, theta=0.25, commit_accept=None, commit_checked=None):
    """Per-record (code, frac) in the reference's check order."""
    out = []
    for r, probs in enumerate(probs_list):
        probs = np.asarray(probs, dtype=np.float64)
        samp_ok, frac = check_sampling(probs, min_sampling_len, p_low, theta)
        if not check_termination(probs, bool(ends_with_eos[r]), int(prompt_len[r]), max_len, eos_prob_floor):
            code = TERMINATION
        elif not samp_ok:
            code = SAMPLING
        elif commit_accept is not None and (commit_checked is None or commit_checked[r]) and not commit_accept[r]:
            code = COMMITMENT
        else:
            code = ACCEPT
        out.append((code, frac))
    return out
