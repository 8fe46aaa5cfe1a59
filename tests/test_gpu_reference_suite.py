"""The reference's own test suite (tests/test_*.py of the reference package,
staged unmodified by oracle/ref_suite.py) run against this package on the
GPU: ``import mpsm`` resolves to paper_1207_0145_b200 and ``mpsm._kernels`` to
its operator layer over the C ABI.  Every reference test must pass except the
ones oracle.ref_suite.EXPECTED_NOT_APPLICABLE lists (the reference's
introsort internals), and those must fail (else the list is stale)."""
import os
import subprocess
import sys
import xml.etree.ElementTree as ET

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import ref_suite  # noqa: E402

pytestmark = pytest.mark.gpu


def test_reference_suite_against_package(tmp_path):
    if not ref_suite.prepare():
        pytest.skip("the reference's tests were not staged (oracle/_ref_tests: built by __graft_entry__.build())")
    xml = tmp_path / "ref.xml"
    env = dict(os.environ, PYTHONDONTWRITEBYTECODE="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", f"--junitxml={xml}",
                        ref_suite.DST], cwd=ref_suite.DST, capture_output=True, text=True, timeout=1200, env=env)
    tree = ET.parse(xml)
    passed, failed, skipped = [], [], []
    for tc in tree.iter("testcase"):
        name = f"{tc.get('file') or tc.get('classname').split('.')[0] + '.py'}::" \
               f"{'::'.join(tc.get('classname').split('.')[1:] + [tc.get('name')])}"
        name = name.replace("::" + tc.get("classname").split(".")[0] + ".py", "")
        kids = {c.tag for c in tc}
        if "failure" in kids or "error" in kids:
            failed.append(name)
        elif "skipped" in kids:
            skipped.append(name)
        else:
            passed.append(name)
    base = lambda n: n.split("[")[0]  # noqa: E731  parametrized ids -> test id
    unexpected = [n for n in failed if base(n) not in ref_suite.EXPECTED_NOT_APPLICABLE]
    stale = [n for n in ref_suite.EXPECTED_NOT_APPLICABLE if n not in {base(f) for f in failed}]
    print(f"reference suite: {len(passed)} passed, {len(failed)} failed "
          f"({len(failed) - len(unexpected)} not applicable), {len(skipped)} skipped")
    assert passed, r.stdout[-3000:] + r.stderr[-3000:]
    assert not unexpected, f"reference tests failing against the package: {unexpected}\n{r.stdout[-6000:]}"
    assert not stale, f"EXPECTED_NOT_APPLICABLE entries that now pass: {stale}"
