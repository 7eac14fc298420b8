"""pytest plugin: installs the swarm adapter in exact mode before the reference's own
test modules are imported.  ``TL_REF_BACKEND=oracle`` (default) uses the exact-mode CPU
oracle as the backend (the adapter's wiring, on any machine); ``TL_REF_BACKEND=gpu`` uses
the product path (``swarm_adapter.GpuBackend``: GPU rounding + SHA-256 chains through the
C ABI).  Used by tests/test_reference_suite.py; not collected on its own."""

import os
import sys

from oracle import exact_oracle as EO
from paper_2505_07291_b200 import swarm_adapter


class _ExactOracleBackend:
    def build_commitments(self, hidden, k):
        return EO.build_commitments(hidden, k)


def pytest_configure(config):
    which = os.environ.get("TL_REF_BACKEND", "oracle")
    if which == "gpu":
        backend = swarm_adapter.GpuBackend()
    elif which == "oracle":
        backend = _ExactOracleBackend()
    else:
        raise ValueError(f"TL_REF_BACKEND={which!r}")
    swarm_adapter.install("exact", backend=backend)
    sys.stderr.write(f"ref_exact_plugin: backend={which}\n")
