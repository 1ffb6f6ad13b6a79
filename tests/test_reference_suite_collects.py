"""API-surface check (build container only): the reference's own test suite
(/root/reference/pkg/tests) collects against this package.  Every module it
imports from `tsdfusion` must resolve to ours with the names it uses, or its
file fails to collect.  The GPU run of the same suite is
scripts/reference_suite.py (profiles/r02_reference_suite.md)."""
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
REF_TESTS = Path("/root/reference/pkg/tests")

pytestmark = [pytest.mark.reference,
              pytest.mark.skipif(not REF_TESTS.is_dir(), reason="needs /root/reference")]


def test_reference_suite_collects_against_this_package(tmp_path):
    code = f"""
import sys, shutil
from pathlib import Path
sys.path.insert(0, {str(ROOT / 'scripts')!r})
import reference_suite as R
stage = Path({str(tmp_path / 'ref_tests')!r})
shutil.copytree(R.REF_TESTS, stage)
R.alias()
import pytest
rc = pytest.main([str(stage), "-q", "--collect-only", "-p", "no:cacheprovider",
                  "--rootdir", str(stage), "-o", "addopts="])
sys.exit(int(rc))
"""
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    tail = [ln for ln in r.stdout.splitlines() if "collected" in ln]
    assert tail and "error" not in tail[-1], tail
    n = int(tail[-1].split()[0])
    assert n >= 200, tail[-1]
