"""`difuser` -> this package: lets the reference's own Python tests
(proj/tests/py/test_smoke.py, run unchanged by tests/test_gpu_scale.py) import
the drop-in under the reference's package name.  Test harness only."""
from paper_2410_14047_b200 import *  # noqa: F401,F403
from paper_2410_14047_b200 import run, run_json  # noqa: F401
