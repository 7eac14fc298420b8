"""Drop this path into the reference's ``swarm`` package without editing it.

The reference binds its commitment function by NAME at three import sites
(no plugin registry):

* ``swarm.worker.rollout.build_commitments``       (rollout.py:51, used at :112)
  and its re-export ``swarm.worker.build_commitments`` (worker/__init__.py:3)
* ``swarm.validator.checks.build_commitments``     (checks.py:27, used at :210-211)
* ``swarm.validator.adversaries.build_commitments`` (adversaries.py:36-42, :312)

``install(mode="exact")`` rebinds all of them to the GPU exact-mode implementation
(byte-identical digests, so the reference's validator works unchanged).

``install(mode="toploc")`` rebinds the prover side to TOPLOC proofs (one 258-byte
proof per ``commit_interval`` rows, hex-encoded into ``RolloutRecord.commitments``
exactly like the digests -- same field, same ``ceil(T/k)`` count, no schema change,
files.py:37,184-186) and wraps ``validate_file`` so that the reference's own check
loop (checks.py:154-215) runs unchanged: for each commitment-checked record, in
the reference's order, the validator-side ``build_commitments`` call verifies the
record's claimed proofs on the GPU against the validator's recomputed hidden
states and returns the claimed proofs when they pass (the reference's list
equality then holds) or an empty list when they fail (reject("commitment")).

``uninstall()`` restores the reference's functions.
"""

from __future__ import annotations

import contextvars
import sys
from dataclasses import dataclass

import numpy as np

from . import codec

TOPLOC_CHUNK = codec.TOPLOC_INTERVAL
_SITES = ("swarm.worker.rollout", "swarm.worker", "swarm.validator.checks", "swarm.validator.adversaries")
_saved: dict = {}
_claimed: contextvars.ContextVar = contextvars.ContextVar("toploc_claimed", default=None)


@dataclass
class GpuBackend:
    """The product path: CUDA kernels through the C ABI (no CPU fallback)."""

    def build_commitments(self, hidden, k):
        from .exact import build_commitments
        return build_commitments(hidden, k)

    def prove(self, hidden_bf16_bits: np.ndarray, k: int) -> list[bytes]:
        from .api import build_proofs
        return build_proofs(hidden_bf16_bits, [0, hidden_bf16_bits.shape[0]], chunk=k)[0]

    def verify(self, hidden_bf16_bits: np.ndarray, proofs: list[bytes], k: int, thresholds) -> bool:
        from .api import verify_proofs
        _, ok = verify_proofs(hidden_bf16_bits, [0, hidden_bf16_bits.shape[0]], [proofs], chunk=k,
                              thresholds=thresholds)
        return bool(ok[0])

    def verify_batch(self, bits: np.ndarray, row_offsets, proofs: np.ndarray, k: int, thresholds) -> np.ndarray:
        """Every record's proofs in one tl_verify: (rows, H) bf16 bits of the records
        concatenated by row_offsets, (n_chunks, 258) proofs -> per-record accept (uint8)."""
        from .api import engine
        vb = engine(chunk=k).verify(bits, row_offsets, proofs, thresholds)
        return vb.rollout_accept.cpu().numpy()

    def record_checks(self, probs, row_offsets, prompt_len, ends_with_eos, rthresholds, commit_accept,
                      commit_checked) -> np.ndarray:
        """tl_record_checks: per-record verdict codes (0 accept, 1 termination, 2 sampling,
        3 commitment) in the reference's order."""
        from .api import record_checks
        v, _, _ = record_checks(probs, row_offsets, prompt_len, ends_with_eos, rthresholds, commit_accept,
                                commit_checked)
        return v.cpu().numpy()


def to_bf16_bits(hidden) -> np.ndarray:
    """(T, H) real array -> bf16 bit patterns (round-to-nearest-even), the precision
    the inference workers commit to."""
    import torch
    t = torch.as_tensor(np.asarray(hidden, dtype=np.float64)).to(torch.bfloat16)
    if t.dim() == 1:
        t = t.reshape(-1, 1)
    return t.view(torch.int16).numpy().view(np.uint16).reshape(t.shape[0], -1)


# --------------------------------------------------------------------------- batched validation
_RECORD_CHECKS = ("accept", "termination", "sampling", "commitment")


def validate_files(blobs, ctx, expected_identities=None, thresholds=None, backend=None, group=None) -> list:
    """``validate_file`` (swarm/validator/checks.py:154-215) over many rollout files, TOPLOC mode.

    The reference runs, per file: schema -> identity -> group size -> seed -> bounds ->
    checkpoint, then per record in order the teacher-forced prefill (schema on error),
    termination, sampling and -- for the q-subsample of ``_commit_sample``
    (checks.py:145-151) -- the commitment check, returning at the first failure.  Here
    the file-level checks and the prefills run per file on the host, exactly as there;
    then EVERY sampled record of every file is verified by one TOPLOC verify call
    (``backend.verify_batch``: one tl_verify), and every record's termination, sampling
    and commitment verdicts come from one ``tl_record_checks`` call, which applies the
    reference's per-record check order.  Each file's verdict is its first failing record
    in record order, with the reference's own detail strings (recomputed on the host for
    that record).  Under torch.distributed with several ranks the files are sharded by
    size over the ranks (``scheduler.shard_by_tokens``) and the verdicts all-gathered, so
    every rank returns the full list.  TOPLOC mode also requires commit_interval == 32."""
    import torch.distributed as dist

    from . import scheduler
    from .api import Thresholds
    backend = backend or GpuBackend()
    th = thresholds or Thresholds()
    blobs = list(blobs)
    ids = list(expected_identities) if expected_identities is not None else [None] * len(blobs)
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if world == 1:
        return _validate_local(blobs, ids, ctx, th, backend)
    rank = dist.get_rank(group)
    lo, hi = scheduler.shard_by_tokens([len(b) for b in blobs], world)[rank]
    local = _validate_local(blobs[lo:hi], ids[lo:hi], ctx, th, backend)
    parts = [None] * world
    dist.all_gather_object(parts, local, group=group)
    return [v for part in parts for v in part]


def _validate_local(blobs, ids, ctx, th, backend) -> list:
    from swarm.policy import sequence_logprobs
    from swarm.tasks import task_for_step
    from swarm.validator.checks import (Verdict, _commit_sample, check_bounds, check_sampling, check_seed,
                                        check_termination)
    from swarm.worker.files import RolloutSchemaError, parse_rollout_file

    from .api import RecordThresholds
    verdicts = [None] * len(blobs)
    files = []  # (file index, file, [record entries])
    for fi, data in enumerate(blobs):
        try:
            f = parse_rollout_file(data)
        except RolloutSchemaError as e:
            verdicts[fi] = Verdict(file_id="unparseable", result="reject", failed_check="schema", details=str(e))
            continue

        def reject(check, details, f=f):
            return Verdict(file_id=f.file_id, result="reject", failed_check=check, details=details,
                           node_address=f.node_address, step=f.step)
        try:  # TOPLOC proofs are defined over 32-token chunks (the reference trusts the header, checks.py:211)
            codec.check_interval(f.commit_interval)
        except codec.ProofFormatError as e:
            verdicts[fi] = reject("schema", str(e))
            continue
        if ids[fi] is not None and ids[fi] != (f.node_address, f.step, f.submission_index):
            verdicts[fi] = reject("schema", "file identity differs from upload slot")
            continue
        if f.group_size != ctx.group_size:
            verdicts[fi] = reject("schema", f"group size {f.group_size} != {ctx.group_size}")
            continue
        if (why := check_seed(f, ctx)) is not None:
            verdicts[fi] = reject("seed", why)
            continue
        if (why := check_bounds(f, ctx)) is not None:
            verdicts[fi] = reject("bounds", why)
            continue
        params = ctx.load_checkpoint(f.checkpoint_version)
        if params is None:
            verdicts[fi] = reject("commitment", f"unknown checkpoint {f.checkpoint_version}")
            continue
        sample = _commit_sample(f, ctx)
        entries = []
        for idx, rec in enumerate(f.records):
            prompt = list(task_for_step(ctx.task(rec.task_id), f.step, ctx.budgets).prompt_tokens)
            try:
                logp, hidden = sequence_logprobs(params, ctx.mcfg, prompt, rec.output_tokens)
            except ValueError as e:  # the reference stops at this record (schema)
                entries.append({"idx": idx, "schema": f"record {idx}: {e}"})
                break
            e = {"idx": idx, "rec": rec, "probs": np.exp(logp), "prompt": prompt, "checked": idx in sample,
                 "proofs": None}
            if e["checked"]:
                try:  # 516-char hex items, ceil(T / 32) of them; a malformed list fails the commitment
                    e["proofs"], _ = codec.decode([rec.commitments], n_tokens=[len(rec.output_tokens)],
                                                  interval=f.commit_interval)
                    e["bits"] = to_bf16_bits(hidden)
                except codec.ProofFormatError:
                    pass
            entries.append(e)
        files.append((fi, f, entries))

    # one TOPLOC verify over every sampled record with well-formed proofs, of every file
    batch = [e for _, _, es in files for e in es if "rec" in e and e["checked"] and e["proofs"] is not None]
    if batch:
        offs = np.concatenate([[0], np.cumsum([e["bits"].shape[0] for e in batch])]).astype(np.int64)
        acc = backend.verify_batch(np.concatenate([e["bits"] for e in batch]), offs,
                                   np.concatenate([e["proofs"] for e in batch]), codec.TOPLOC_INTERVAL, th)
        for e, a in zip(batch, acc):
            e["commit_ok"] = bool(a)
    # one record-checks call: termination, sampling, commitment in the reference's order
    recs = [e for _, _, es in files for e in es if "rec" in e]
    codes = []
    if recs:
        offs = np.concatenate([[0], np.cumsum([len(e["probs"]) for e in recs])]).astype(np.int64)
        rth = RecordThresholds(max_len=ctx.mcfg.max_len, min_sampling_len=ctx.min_sampling_len,
                               eos_prob_floor=ctx.eos_prob_floor, p_low=ctx.p_low, theta=ctx.theta)
        codes = backend.record_checks(
            np.concatenate([e["probs"] for e in recs]), offs, [len(e["prompt"]) for e in recs],
            [bool(e["rec"].output_tokens) and e["rec"].output_tokens[-1] == ctx.mcfg.eos_id for e in recs], rth,
            np.array([e.get("commit_ok", False) for e in recs], dtype=np.uint8),
            np.array([e["checked"] for e in recs], dtype=np.uint8))
    for e, code in zip(recs, codes):
        e["code"] = int(code)
    for fi, f, entries in files:
        v = Verdict(file_id=f.file_id, result="accept", node_address=f.node_address, step=f.step)
        for e in entries:
            check = "schema" if "schema" in e else _RECORD_CHECKS[e["code"]]
            if check == "accept":
                continue
            idx = e["idx"]
            if check == "schema":
                details = e["schema"]
            elif check == "termination":
                details = f"record {idx}: {check_termination(e['rec'], e['probs'], len(e['prompt']), ctx)}"
            elif check == "sampling":
                details = f"record {idx}: {check_sampling(e['rec'], e['probs'], ctx)}"
            else:
                details = f"record {idx}: digest mismatch"
            v = Verdict(file_id=f.file_id, result="reject", failed_check=check, details=details,
                        node_address=f.node_address, step=f.step)
            break
        verdicts[fi] = v
    return verdicts


def _modules():
    import importlib
    return {name: importlib.import_module(name) for name in _SITES}


def install(mode: str = "exact", thresholds=None, backend=None, batched: bool = True) -> None:
    """Rebind the reference's ``build_commitments`` sites (and, in TOPLOC mode,
    ``validate_file``) to this package.  TOPLOC mode with ``batched`` (the default) routes
    ``validate_file`` through ``validate_files`` (every sampled record of the file in one
    verify call); ``batched=False`` wraps the reference's own ``validate_file`` loop and
    verifies record by record from inside it."""
    from .api import Thresholds
    if mode not in ("exact", "toploc"):
        raise ValueError("mode must be 'exact' or 'toploc'")
    uninstall()
    backend = backend or GpuBackend()
    th = thresholds or Thresholds()
    mods = _modules()
    for name, mod in mods.items():
        _saved[(name, "build_commitments")] = mod.build_commitments
    checks = mods["swarm.validator.checks"]
    _saved[("swarm.validator.checks", "validate_file")] = checks.validate_file
    import swarm.validator as validator_pkg
    _saved[("swarm.validator", "validate_file")] = validator_pkg.validate_file
    # swarm/node.py:30 binds validate_file by name at import: rebind it when it is already
    # loaded (a later import reads the rebound swarm.validator attribute)
    node = sys.modules.get("swarm.node")
    if node is not None and hasattr(node, "validate_file"):
        _saved[("swarm.node", "validate_file")] = node.validate_file

    if mode == "exact":
        def exact_commitments(hidden, k=32):
            return backend.build_commitments(hidden, k)
        for mod in mods.values():
            mod.build_commitments = exact_commitments
        return

    def prove_commitments(hidden, k=32):
        if k < 1:
            raise ValueError("interval must be >= 1")
        return backend.prove(to_bf16_bits(hidden), k)

    def verify_commitments(hidden, k=32):
        queue = _claimed.get()
        if queue is None:
            # only the wrapped validate_file sets the claimed proofs; re-proving here would
            # turn TOPLOC's tolerance back into byte equality (honest workers rejected)
            raise RuntimeError("TOPLOC validator commitment check called outside the installed "
                               "validate_file (a module bound the original validate_file before install())")
        claimed = queue.pop(0)
        try:  # 516-char hex items, ceil(T / 32) of them (codec.py, files.py:184-186)
            arr, _ = codec.decode([claimed], n_tokens=[len(hidden)], interval=k)
        except codec.ProofFormatError:
            return []
        proofs = [arr[j].tobytes() for j in range(arr.shape[0])]
        return proofs if backend.verify(to_bf16_bits(hidden), proofs, k, th) else []

    orig_validate = _saved[("swarm.validator.checks", "validate_file")]

    def validate_file_batched(data, ctx, expected_identity=None):
        return validate_files([data], ctx, [expected_identity], th, backend)[0]

    def validate_file(data, ctx, expected_identity=None):
        from swarm.validator.checks import Verdict, _commit_sample
        from swarm.worker.files import RolloutSchemaError, parse_rollout_file
        try:
            f = parse_rollout_file(data)
            queue = [list(f.records[i].commitments) for i in sorted(_commit_sample(f, ctx))]
        except (RolloutSchemaError, Exception):
            f, queue = None, []
        if f is not None:
            # TOPLOC proofs are defined over 32-token chunks; the reference trusts the
            # header's interval (checks.py:211), TOPLOC mode enforces it
            try:
                codec.check_interval(f.commit_interval)
            except codec.ProofFormatError as e:
                return Verdict(file_id=f.file_id, result="reject", failed_check="schema", details=str(e),
                               node_address=f.node_address, step=f.step)
        token = _claimed.set(queue)
        try:
            return orig_validate(data, ctx, expected_identity)
        finally:
            _claimed.reset(token)

    mods["swarm.worker.rollout"].build_commitments = prove_commitments
    mods["swarm.worker"].build_commitments = prove_commitments
    mods["swarm.validator.adversaries"].build_commitments = prove_commitments
    checks.build_commitments = verify_commitments
    vf = validate_file_batched if batched else validate_file
    checks.validate_file = vf
    validator_pkg.validate_file = vf
    if ("swarm.node", "validate_file") in _saved:
        node.validate_file = vf


def uninstall() -> None:
    if not _saved:
        return
    import importlib
    for (name, attr), fn in _saved.items():
        setattr(importlib.import_module(name), attr, fn)
    _saved.clear()
