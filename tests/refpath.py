"""Where the reference (swarm-rl) lives for the tests that run it: /root/reference/pkg in
the build container, else the install tools/install_reference.sh makes under
baseline/_ref (git-ignored; it travels to the GPU box with the gpurun snapshot)."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_CANDIDATES = (
    ("/root/reference/pkg/src", "/root/reference/pkg/tests"),
    (os.path.join(ROOT, "baseline", "_ref"), os.path.join(ROOT, "baseline", "_ref", "swarm_ref_tests")),
)


def ref_src():
    """Directory holding the importable ``swarm`` package, or None."""
    for src, _ in _CANDIDATES:
        if os.path.isfile(os.path.join(src, "swarm", "__init__.py")):
            return src
    return None


def ref_tests():
    """Directory holding the reference's own test files, or None."""
    for src, tests in _CANDIDATES:
        if os.path.isfile(os.path.join(src, "swarm", "__init__.py")) and os.path.isfile(
                os.path.join(tests, "test_validator.py")):
            return tests
    return None


def add_ref_to_path():
    src = ref_src()
    if src and src not in sys.path:
        sys.path.append(src)
    return src
