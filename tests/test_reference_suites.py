"""The reference's own test suites, unchanged, against this package.

tests/dropsim_alias.py registers `paper_2412_18169_b200` under the name
`dropsim`; pytest then runs /root/reference/pkg/tests/*.py (all but
test_cli.py, whose matplotlib front end is out of scope) in model mode:
memory, planner, exchange, engine, formulation, cost model, metrics, trace
I/O, config -- and the 8-criterion acceptance checklist
(pkg/tests/test_acceptance.py).  Skipped where /root/reference is absent
(the GPU box); nothing is copied from the reference.
"""

import os
import re
import subprocess
import sys

import pytest

REF = "/root/reference/pkg"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "tests")), reason="reference not present")
def test_reference_suites_pass_against_this_package():
    files = sorted(f for f in os.listdir(os.path.join(REF, "tests"))
                   if f.startswith("test_") and f.endswith(".py") and f != "test_cli.py")
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1",
               PYTHONPATH=os.pathsep.join([ROOT, os.path.join(ROOT, "tests")]))
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "dropsim_alias",
                          "-p", "no:cacheprovider", *[os.path.join("tests", f) for f in files]],
                         cwd=REF, env=env, capture_output=True, text=True, timeout=900)
    tail = res.stdout[-2000:]
    assert res.returncode == 0, tail
    m = re.search(r"(\d+) passed", tail)
    assert m and int(m.group(1)) >= 130, tail
