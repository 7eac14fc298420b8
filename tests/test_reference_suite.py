"""The reference's own commitment and validator tests (pkg/tests/test_rollout.py,
pkg/tests/test_validator.py), unmodified, with this package's adapter installed in exact
mode ('what the B200 build reuses').  CPU; skipped where the reference is not
present (the GPU box)."""

import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/pkg"


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")), reason="reference not present")
def test_reference_rollout_and_validator_suites_pass_through_the_adapter():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(REF, "src"), ROOT, os.path.join(ROOT, "tests")])
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "ref_exact_plugin", "-p", "no:cacheprovider",
                        "--rootdir", REF, os.path.join(REF, "tests", "test_rollout.py"),
                        os.path.join(REF, "tests", "test_validator.py")],
                       cwd="/tmp", env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert " passed" in r.stdout and "failed" not in r.stdout


def test_plugin_rebinds_every_site():
    """Without the reference there is nothing to rebind; with it, the plugin's install
    reaches the three import sites (rollout.py:51, checks.py:27, adversaries.py:36-42)."""
    if not os.path.isdir(os.path.join(REF, "src")):
        pytest.skip("reference not present")
    if os.path.join(REF, "src") not in sys.path:
        sys.path.append(os.path.join(REF, "src"))
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
