"""GPU: every kernel entry point under the bounds-checked build (device asserts on the hot
kernels' shared / global indices; `python -m paper_2603_01122_b200.build --checked`).

compute-sanitizer is not available on this GPU pool, so the checked build is how the
suite looks for out-of-range accesses: tools/sanitize_run.py drives K1/K2 (all modes,
window and global-histogram paths, chunked horizons)/K3 and the f-row kernels at small
sizes in a subprocess that loads the checked library; any failed assert aborts it.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2603_01122_b200", "_lib", "checked", "libgridcast_b200.so")


def test_all_entry_points_under_bounds_checks():
    if not os.path.exists(CHECKED):
        pytest.skip("checked build absent (python -m paper_2603_01122_b200.build --checked)")
    env = dict(os.environ, GC_LIB_PATH=CHECKED)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")], env=env,
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0 and "all entry points ran" in out.stdout, (out.stdout[-2000:], out.stderr[-4000:])
    assert "Assertion" not in out.stderr
