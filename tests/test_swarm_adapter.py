"""The swarm adapter against the reference's own validator (swarm/validator/checks.py:154-215,
swarm/validator/adversaries.py), where the reference package is importable
(/root/reference/pkg/src here, baseline/_ref on the GPU box: tests/refpath.py).

Every test runs with two backends: the CPU oracle (wiring through the reference's real
control flow, on any machine) and the product GPU path (``GpuBackend``: the CUDA kernels
through the C ABI, ``-m gpu``)."""

import numpy as np
import pytest

from refpath import add_ref_to_path

add_ref_to_path()
swarm = pytest.importorskip("swarm")

from oracle import exact_oracle as EO  # noqa: E402
from oracle import toploc_oracle as TO  # noqa: E402
from paper_2505_07291_b200 import swarm_adapter  # noqa: E402
from paper_2505_07291_b200.api import Thresholds  # noqa: E402


class OracleBackend:
    def build_commitments(self, hidden, k):
        return EO.build_commitments(hidden, k)

    def prove(self, bits, k):
        return TO.build_proofs(bits, [0, bits.shape[0]], C=k)[0]

    def verify(self, bits, proofs, k, th):
        _, ok = TO.verify_proofs(bits, [0, bits.shape[0]], [proofs], C=k,
                                 th=TO.Thresholds(th.max_exp_mismatch, th.max_mant_mean, th.max_mant_median))
        return ok[0]


@pytest.fixture(params=["oracle", pytest.param("gpu", marks=pytest.mark.gpu)])
def backend(request):
    """A fresh backend factory: the oracle stand-in or the product GPU path."""
    if request.param == "oracle":
        return OracleBackend
    return swarm_adapter.GpuBackend


def fixtures():
    from swarm.config import TOY_MODEL
    from swarm.keys import SigningKey
    from swarm.policy import init_params
    from swarm.tasks import generate_dataset
    from swarm.validator import CheckContext
    from swarm.validator.adversaries import Forge
    dataset = generate_dataset(seed=10, n=64)
    params = init_params(TOY_MODEL, seed=2, scale=1.0)
    stale = params.copy()
    rng = np.random.default_rng(3)
    for a in stale.arrays():
        a += rng.normal(0, 1e-3, a.shape)
    other = init_params(TOY_MODEL, seed=77, scale=1.0)
    forge = Forge(params=params, stale_params=stale, other_params=other, mcfg=TOY_MODEL, dataset=dataset,
                  key=SigningKey.from_seed(7, 0), checkpoint_version=5)
    ctx = CheckContext(mcfg=TOY_MODEL, dataset=dataset, alpha=0.01, budgets=(8, 16, 24, 32), group_size=4,
                       p_low=0.005, load_checkpoint=lambda v: {5: params, 2: stale}.get(v))
    return forge, ctx


@pytest.fixture
def adapter():
    yield swarm_adapter
    swarm_adapter.uninstall()


def validate(blob, ctx):
    import swarm.validator.checks as checks
    return checks.validate_file(blob, ctx)


def test_exact_mode_is_byte_identical_and_keeps_verdicts(adapter, backend):
    import swarm.worker.rollout as rollout
    forge, ctx = fixtures()
    orig = rollout.build_commitments
    h = np.random.default_rng(0).normal(size=(70, 8))
    adapter.install("exact", backend=backend())
    assert rollout.build_commitments is not orig
    assert rollout.build_commitments(h) == orig(h)
    for step in (1, 2):
        assert validate(forge.honest(step, 0), ctx).result == "accept"
        v = validate(forge.generate("wrong-model", step, 0), ctx)
        assert (v.result, v.failed_check) == ("reject", "commitment")
    adapter.uninstall()
    assert rollout.build_commitments is orig


def test_toploc_mode_wire_format(adapter, backend):
    from swarm.worker.files import parse_rollout_file
    forge, ctx = fixtures()
    adapter.install("toploc", backend=backend())
    f = parse_rollout_file(forge.honest(3, 0))
    for rec in f.records:
        assert len(rec.commitments) == -(-len(rec.output_tokens) // f.commit_interval)
        assert all(len(c) == 2 * 258 for c in rec.commitments)


@pytest.mark.parametrize("attack", ["malformed-file", "cherry-picked-prompt", "forged-reward", "early-eos",
                                    "token-substitution"])
def test_toploc_mode_keeps_reference_check_order(adapter, attack, backend):
    from swarm.validator.adversaries import EXPECTED_CHECK
    forge, ctx = fixtures()
    adapter.install("toploc", backend=backend())
    assert validate(forge.honest(2, 0), ctx).result == "accept"
    v = validate(forge.generate(attack, 2, 0), ctx)
    assert (v.result, v.failed_check) == ("reject", EXPECTED_CHECK[attack])


def test_toploc_mode_commitment_verdicts(adapter, backend):
    """Honest files pass; a tampered proof and an unrelated model are rejected at
    the commitment check.  The reference's 'wrong-model' forgery (a checkpoint
    within 1e-3 of the claimed one) is within TOPLOC's tolerance at the default
    thresholds (accept) and rejected at exact thresholds."""
    from swarm.worker.files import build_rollout_file, parse_rollout_file
    forge, ctx = fixtures()
    adapter.install("toploc", backend=backend())
    for step in (1, 2, 3):
        assert validate(forge.honest(step, 0), ctx).result == "accept"
    f = parse_rollout_file(forge.honest(4, 0))
    p = bytearray(bytes.fromhex(f.records[1].commitments[0]))
    p[0:2] = (65479).to_bytes(2, "big")                    # wrong modulus -> garbage evaluations
    f.records[1].commitments[0] = bytes(p).hex()
    v = validate(build_rollout_file(f, forge.key), ctx)
    assert (v.result, v.failed_check) == ("reject", "commitment") and "record 1" in v.details
    wm = forge.generate("wrong-model", 1, 0)
    assert validate(wm, ctx).result == "accept"
    adapter.install("toploc", thresholds=Thresholds(0, 0.0, 0.0), backend=backend())
    v = validate(wm, ctx)
    assert (v.result, v.failed_check) == ("reject", "commitment")


def test_toploc_mode_enforces_commit_interval(adapter, backend):
    from swarm.worker.files import build_rollout_file, parse_rollout_file
    forge, ctx = fixtures()
    adapter.install("toploc", backend=backend())
    f = parse_rollout_file(forge.honest(2, 0))
    f.commit_interval = 16
    for rec in f.records:
        rec.commitments = rec.commitments + rec.commitments        # right count for k = 16 is irrelevant
        rec.commitments = rec.commitments[:-(-len(rec.output_tokens) // 16)] if len(rec.commitments) > \
            -(-len(rec.output_tokens) // 16) else rec.commitments + [rec.commitments[0]] * (
                -(-len(rec.output_tokens) // 16) - len(rec.commitments))
    v = validate(build_rollout_file(f, forge.key), ctx)
    assert (v.result, v.failed_check) == ("reject", "schema") and "commit_interval" in v.details


def test_toploc_mode_rebinds_an_already_imported_node(adapter, backend):
    """swarm/node.py:30 binds validate_file by name at import.  When the node module was
    imported before install(), its binding is rebound too (and restored afterwards), so
    the node's validator runs the TOPLOC check instead of the original digest compare."""
    import swarm.node as node
    import swarm.validator.checks as checks
    orig = node.validate_file
    forge, ctx = fixtures()
    adapter.install("toploc", backend=backend())
    assert node.validate_file is checks.validate_file and node.validate_file is not orig
    assert node.validate_file(forge.honest(2, 0), ctx).result == "accept"
    adapter.uninstall()
    assert node.validate_file is orig


def test_toploc_validator_commitments_outside_validate_file_raise(adapter, backend):
    """The validator-side commitment function only has claimed proofs inside the wrapped
    validate_file; anywhere else it raises instead of silently re-proving (which would
    turn TOPLOC's tolerance back into byte equality)."""
    import swarm.validator.checks as checks
    adapter.install("toploc", backend=backend())
    with pytest.raises(RuntimeError, match="outside the installed validate_file"):
        checks.build_commitments(np.zeros((32, 8)), 32)


@pytest.mark.parametrize("q", [1.0, 0.5])
def test_toploc_mode_honours_the_commit_q_subsample(adapter, backend, q):
    """checks.py:145-151: with commit_q < 1 only the q-subsample of records is
    commitment-checked.  A record whose first proof is tampered rejects the file at the
    commitment check iff the reference's own _commit_sample picks it."""
    from swarm.validator.checks import _commit_sample
    from swarm.worker.files import build_rollout_file, parse_rollout_file
    forge, ctx = fixtures()
    ctx.commit_q, ctx.q_seed = q, 5
    adapter.install("toploc", backend=backend())
    blob = forge.honest(3, 0)
    assert validate(blob, ctx).result == "accept"
    f0 = parse_rollout_file(blob)
    sample = _commit_sample(f0, ctx)
    assert (len(sample) == len(f0.records)) == (q >= 1.0) and len(sample) > 0
    for i in range(len(f0.records)):
        f = parse_rollout_file(blob)
        p = bytearray(bytes.fromhex(f.records[i].commitments[0]))
        p[0:2] = (65479).to_bytes(2, "big")
        f.records[i].commitments[0] = bytes(p).hex()
        v = validate(build_rollout_file(f, forge.key), ctx)
        if i in sample:
            assert (v.result, v.failed_check) == ("reject", "commitment") and f"record {i}" in v.details
        else:
            assert v.result == "accept", i
