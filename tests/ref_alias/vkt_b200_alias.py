"""pytest plugin (``-p vkt_b200_alias``): make ``import vkt`` resolve to this
package's reference-compatible namespace (paper_2203_10213_b200.vkt), so the
reference's own test files run unmodified against the B200 path.  Loaded as a
plugin, it is in place before the reference's conftest.py imports ``vkt``."""

import importlib
import sys

_SUBMODULES = ("errors", "ops", "ops.filters", "ops.core")

facade = importlib.import_module("paper_2203_10213_b200.vkt")
sys.modules["vkt"] = facade
for _name in _SUBMODULES:
    sys.modules[f"vkt.{_name}"] = importlib.import_module(f"paper_2203_10213_b200.vkt.{_name}")


# Collection scaffolding, not API: test_ops_core.py parametrizes its
# (out-of-scope, deselected) arithmetic tests over ``vkt.ArithmeticOp`` at
# import time (test_ops_core.py:242), so the module only imports if the enum
# exists.  The package does not implement voxel arithmetic;
# this enum lists the reference's members (ops/core.py:268-273) for
# collection and nothing calls it.
if not hasattr(facade, "ArithmeticOp"):
    from enum import Enum

    facade.ArithmeticOp = Enum("ArithmeticOp", {"SUM": "sum", "DIFF": "diff", "PROD": "prod",
                                                "QUOT": "quot", "ABS_DIFF": "absdiff"})


def pytest_report_header(config):
    return f"vkt -> {facade.__name__} ({facade.__file__})"
