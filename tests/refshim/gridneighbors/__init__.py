"""Alias package: ``gridneighbors`` -> ``paper_2004_02290_b200`` (TEST
INFRASTRUCTURE ONLY), so the reference's own test suite
(pkg/tests, staged under baseline/_ref/pkg/tests by
tools/stage_reference_tests.sh) imports the drop-in instead of the
reference.  Submodules map to their counterparts: ``bench`` is
``runbench`` (the run_bench harness); the rest share names."""
import sys

import paper_2004_02290_b200 as _pkg
from paper_2004_02290_b200 import *  # noqa: F401,F403
from paper_2004_02290_b200 import __all__  # noqa: F401
from paper_2004_02290_b200 import baselines, core, datasets, explore, grid, predict, runbench

for _name, _mod in {"baselines": baselines, "core": core, "datasets": datasets, "explore": explore,
                    "grid": grid, "predict": predict, "bench": runbench}.items():
    sys.modules[__name__ + "." + _name] = _mod
    globals()[_name] = _mod
__version__ = _pkg.__version__
