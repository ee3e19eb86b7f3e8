"""conftest for running the reference package's OWN test suite against this
package (tools/run_reference_suite.sh): `micromech` and its submodules are
aliased to paper_2010_06697_b200, so every `from micromech... import ...` in
the reference tests binds our names and every solve / projection / local step
/ stability call runs the sm_100a library (there is no CPU fallback: without
a GPU those tests raise "no CUDA device")."""

import importlib
import os
import sys

sys.path.insert(0, os.environ.get("MM_REPO", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import paper_2010_06697_b200 as _pkg  # noqa: E402

sys.modules["micromech"] = _pkg
for _sub in ("grid", "projection", "solver", "stability", "errors", "materials", "scenarios"):
    sys.modules["micromech." + _sub] = importlib.import_module("paper_2010_06697_b200." + _sub)


def pytest_terminal_summary(terminalreporter):
    """Name the native library the run actually mapped (/proc/self/maps)."""
    try:
        with open("/proc/self/maps") as f:
            libs = sorted({ln.split()[-1] for ln in f if "libmm_admm" in ln})
    except OSError:
        libs = []
    terminalreporter.write_line(f"native library loaded: {libs or 'none'}")
