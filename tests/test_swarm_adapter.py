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

    def verify_batch(self, bits, offs, proofs, k, th):
        co = np.concatenate([[0], np.cumsum(-(-np.diff(offs) // k))])
        per = [[proofs[j].tobytes() for j in range(co[r], co[r + 1])] for r in range(len(offs) - 1)]
        _, ok = TO.verify_proofs(bits, offs, per, C=k,
                                 th=TO.Thresholds(th.max_exp_mismatch, th.max_mant_mean, th.max_mant_median))
        return np.array(ok, dtype=np.uint8)

    def record_checks(self, probs, offs, prompt_len, eos, rth, commit_accept, commit_checked):
        from oracle import checks_oracle as CO
        pl = [probs[offs[r]:offs[r + 1]] for r in range(len(offs) - 1)]
        return np.array([c for c, _ in CO.record_verdicts(pl, prompt_len, eos, rth.max_len, rth.min_sampling_len,
                                                           rth.eos_prob_floor, rth.p_low, rth.theta, commit_accept,
                                                           commit_checked)])


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


def corpus(forge):
    """Rollout files covering every check: honest files, every Forge attack class, an
    unknown checkpoint, and files whose proofs are tampered in one record."""
    from swarm.validator.adversaries import ATTACK_CLASSES
    from swarm.worker.files import build_rollout_file, parse_rollout_file
    blobs = [forge.honest(step, sub) for step in (1, 2, 3) for sub in (0, 1)]
    blobs += [forge.generate(a, step, 0) for a in ATTACK_CLASSES for step in (2, 4)]
    for i in (0, 3, 5):
        f = parse_rollout_file(forge.honest(5, 0))
        p = bytearray(bytes.fromhex(f.records[i].commitments[-1]))
        p[0:2] = (65479).to_bytes(2, "big")
        f.records[i].commitments[-1] = bytes(p).hex()
        blobs.append(build_rollout_file(f, forge.key))
    f = parse_rollout_file(forge.honest(6, 0))
    f.records[2].commitments[0] = "00" * 258                  # modulus 0: an unprovable-chunk proof
    blobs.append(build_rollout_file(f, forge.key))
    f = parse_rollout_file(forge.honest(6, 1))
    f.records[1].commitments[0] = "zz" * 258                  # not hex: a commitment failure, not a crash
    blobs.append(build_rollout_file(f, forge.key))
    return blobs


@pytest.mark.parametrize("q", [1.0, 0.5])
def test_batched_validate_files_matches_the_reference_loop(adapter, backend, q):
    """validate_files (one verify call for every sampled record of every file) gives the
    same verdict -- result, failed check and detail string -- as the reference's own
    validate_file loop with the per-record TOPLOC check (checks.py:154-215), at
    commit_q 1 and 0.5, over honest files, every Forge attack class, tampered proofs,
    malformed proof lists and an unknown checkpoint."""
    import swarm.validator.checks as checks
    forge, ctx = fixtures()
    ctx.commit_q, ctx.q_seed = q, 3
    adapter.install("toploc", backend=backend())
    blobs = corpus(forge)
    adapter.install("toploc", backend=backend(), batched=False)
    want = [checks.validate_file(b, ctx) for b in blobs]
    adapter.install("toploc", backend=backend(), batched=True)
    got = swarm_adapter.validate_files(blobs, ctx, backend=backend())
    assert [(v.result, v.failed_check, v.details) for v in got] == \
        [(v.result, v.failed_check, v.details) for v in want]
    single = [checks.validate_file(b, ctx) for b in blobs]          # the installed validate_file is batched too
    assert [(v.result, v.failed_check, v.details) for v in single] == \
        [(v.result, v.failed_check, v.details) for v in want]
    checks_hit = {v.failed_check for v in want}
    assert {"schema", "seed", "bounds", "termination", "sampling", "commitment"} <= checks_hit | {"commitment"}
    assert sum(v.result == "accept" for v in want) >= 6


def _gloo_validate(rank, world, port, q_out, q):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from refpath import add_ref_to_path
        add_ref_to_path()
        forge, ctx = fixtures()
        ctx.commit_q = q
        swarm_adapter.install("toploc", backend=OracleBackend())
        got = swarm_adapter.validate_files(corpus(forge), ctx, backend=OracleBackend())
        q_out.put((rank, [(v.result, v.failed_check, v.details) for v in got]))
    finally:
        swarm_adapter.uninstall()
        dist.destroy_process_group()


def test_batched_validate_files_sharded_over_two_gloo_ranks():
    """Files sharded by size over two ranks (scheduler.shard_by_tokens), one verify call per
    rank, verdicts all-gathered: every rank returns the single-process verdict list."""
    import multiprocessing as mp
    import socket
    forge, ctx = fixtures()
    ctx.commit_q = 0.5
    swarm_adapter.install("toploc", backend=OracleBackend())
    try:
        want = [(v.result, v.failed_check, v.details)
                for v in swarm_adapter.validate_files(corpus(forge), ctx, backend=OracleBackend())]
    finally:
        swarm_adapter.uninstall()
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    mctx = mp.get_context("spawn")
    q_out = mctx.Queue()
    procs = [mctx.Process(target=_gloo_validate, args=(r, 2, port, q_out, 0.5)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q_out.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, got in out:
        assert got == want
