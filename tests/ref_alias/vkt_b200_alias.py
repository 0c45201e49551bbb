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


def pytest_report_header(config):
    return f"vkt -> {facade.__name__} ({facade.__file__})"
