"""pytest plugin (CPU): installs the swarm adapter in exact mode before the reference's own
test modules are imported, with the exact-mode oracle standing in for the GPU path (the
GPU path's byte-identity is tested in tests/test_gpu_exact.py).  Used by
tests/test_reference_suite.py; not collected on its own."""

from oracle import exact_oracle as EO
from paper_2505_07291_b200 import swarm_adapter


class _ExactOracleBackend:
    def build_commitments(self, hidden, k):
        return EO.build_commitments(hidden, k)


def pytest_configure(config):
    swarm_adapter.install("exact", backend=_ExactOracleBackend())
