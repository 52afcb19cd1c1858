"""pytest plugin: run the reference's OWN test files (baseline/_ref/parmcmc_tests, copied
from /root/reference/pkg/tests by __graft_entry__.install_reference) against the drop-in.

Every `parmcmc` module name resolves to the matching paper_1310_1537_b200 module, so
`from parmcmc import glm` / `from parmcmc.ising import gibbs_sweep` in the reference's
tests import the B200 implementation (module aliasing; the reference package itself is
not on sys.path).  Used by tests/test_gpu_reference_suite.py.
"""

import importlib
import sys

_SUBMODULES = ("glm", "sampler", "ising", "hb", "rng", "perf", "parallel", "instrumentation", "cli")


def _install():
    pkg = importlib.import_module("paper_1310_1537_b200")
    sys.modules["parmcmc"] = pkg
    for name in _SUBMODULES:
        sys.modules[f"parmcmc.{name}"] = importlib.import_module(f"paper_1310_1537_b200.{name}")


_install()
