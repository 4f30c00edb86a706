"""pytest plugin: run the reference's own test files against the B200 path.

    B200_PLUGIN_MODE=kernel|execute python -m pytest -p integration.plugin \
        baseline/_ref/tests/test_kernels.py baseline/_ref/tests/test_attention.py ...

(baseline/_ref is the unmodified reference installed by
tools/install_reference.sh, its tests copied beside it.) At the end the
plugin prints how many calls went through the B200 path."""
from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
for p in (ROOT / "baseline" / "_ref", ROOT):
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))


def pytest_configure(config):
    from integration import prefixdec_b200
    prefixdec_b200.install(os.environ.get("B200_PLUGIN_MODE", "kernel"))
    # the executor module's name binding: tests import `execute` from there
    import prefixdec.executor  # noqa: F401


def pytest_terminal_summary(terminalreporter):
    from integration.prefixdec_b200 import CALLS
    terminalreporter.write_line(f"B200 plugin calls: {CALLS}")
