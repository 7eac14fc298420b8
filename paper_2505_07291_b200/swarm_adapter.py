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


def to_bf16_bits(hidden) -> np.ndarray:
    """(T, H) real array -> bf16 bit patterns (round-to-nearest-even), the precision
    the inference workers commit to."""
    import torch
    t = torch.as_tensor(np.asarray(hidden, dtype=np.float64)).to(torch.bfloat16)
    if t.dim() == 1:
        t = t.reshape(-1, 1)
    return t.view(torch.int16).numpy().view(np.uint16).reshape(t.shape[0], -1)


def _modules():
    import importlib
    return {name: importlib.import_module(name) for name in _SITES}


def install(mode: str = "exact", thresholds=None, backend=None) -> None:
    """Rebind the reference's ``build_commitments`` sites (and, in TOPLOC mode,
    ``validate_file``) to this package."""
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
    checks.validate_file = validate_file
    validator_pkg.validate_file = validate_file
    if ("swarm.node", "validate_file") in _saved:
        node.validate_file = validate_file


def uninstall() -> None:
    if not _saved:
        return
    import importlib
    for (name, attr), fn in _saved.items():
        setattr(importlib.import_module(name), attr, fn)
    _saved.clear()
