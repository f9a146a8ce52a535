"""Run the reference's own mcx test file against the drop-in ``nlrom.mcx``.

``tests/golden/ref_tests/test_mcx.py`` is the unmodified reference test file
(/root/reference/pkg/tests/test_mcx.py, 33 tests), committed as test infrastructure. It
imports ``from nlrom import mcx``; here ``nlrom`` resolves to this repo's package
(``nlrom/__init__.py`` -> ``paper_2102_11026_b200``), so every reference test exercises
the product implementation (the import swap SURVEY.md §7 step 2 asks for)."""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_mcx_suite_against_dropin():
    env = dict(os.environ, PYTHONPATH=ROOT)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                        os.path.join(ROOT, "tests", "golden", "ref_tests", "test_mcx.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "33 passed" in r.stdout, r.stdout[-2000:]
    # and the module under test is the product, not the reference
    probe = subprocess.run([sys.executable, "-c", "from nlrom import mcx; print(mcx.__file__)"],
                           cwd=ROOT, env=env, capture_output=True, text=True, timeout=120)
    assert "paper_2102_11026_b200" in probe.stdout, probe.stdout + probe.stderr
