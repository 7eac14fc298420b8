"""The reference's own commitment and validator tests (pkg/tests/test_rollout.py,
pkg/tests/test_validator.py), unmodified, with this package's adapter installed in exact
mode ('what the B200 build reuses').

Two backends: the exact-mode CPU oracle (any machine) and the product GPU exact path
(``-m gpu``: GPU rounding plus the SHA-256 chains, through the C ABI).  The reference is
found at /root/reference/pkg here or under baseline/_ref on the GPU box
(tools/install_reference.sh; tests/refpath.py)."""

import os
import subprocess
import sys

import pytest

from refpath import ref_src, ref_tests

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC, TESTS = ref_src(), ref_tests()


@pytest.mark.skipif(TESTS is None, reason="reference not present (run tools/install_reference.sh)")
@pytest.mark.parametrize("backend", ["oracle", pytest.param("gpu", marks=pytest.mark.gpu)])
def test_reference_rollout_and_validator_suites_pass_through_the_adapter(backend):
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([SRC, ROOT, os.path.join(ROOT, "tests")])
    env["TL_REF_BACKEND"] = backend
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "ref_exact_plugin", "-p", "no:cacheprovider",
                        "--rootdir", os.path.dirname(TESTS), os.path.join(TESTS, "test_rollout.py"),
                        os.path.join(TESTS, "test_validator.py")],
                       cwd="/tmp", env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout
    assert f"ref_exact_plugin: backend={backend}" in r.stdout + r.stderr


def test_plugin_rebinds_every_site():
    """Without the reference there is nothing to rebind; with it, the plugin's install
    reaches the three import sites (rollout.py:51, checks.py:27, adversaries.py:36-42)."""
    if SRC is None:
        pytest.skip("reference not present")
    if SRC not in sys.path:
        sys.path.append(SRC)
    import importlib
    from paper_2505_07291_b200 import swarm_adapter
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    plugin = importlib.import_module("ref_exact_plugin")
    try:
        plugin.pytest_configure(None)
        for name in ("swarm.worker.rollout", "swarm.worker", "swarm.validator.checks", "swarm.validator.adversaries"):
            fn = importlib.import_module(name).build_commitments
            assert fn.__module__ == "paper_2505_07291_b200.swarm_adapter", name
    finally:
        swarm_adapter.uninstall()
