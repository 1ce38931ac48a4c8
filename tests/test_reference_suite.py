"""Run the REFERENCE's own tests (/root/reference/pkg/tests) against this
package through the `migsim` import alias.  Only in the build container (the
reference tree does not travel to the GPU box).

Deselected, as outside the one-to-many path: Dynamic-MIG
(`test_dm_*`, 6 of 8 also fail on the reference itself), reconfiguration
economics (`test_merge_*`, `test_plan_*`, `test_pack_*`) and the
discrete-event simulator engine (test_simcore.py beyond `estimate_jct`).
"""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

OUT_OF_SCOPE = ("test_dm_ or test_merge_ or test_plan_ or test_pack_ or "
                "(test_simcore and not test_estimate and not test_multi_overhead)")


@pytest.mark.skipif(not os.path.isdir(REF_TESTS), reason="reference tree not mounted")
def test_reference_hot_path_tests_pass_on_this_package(tmp_path):
    files = [os.path.join(REF_TESTS, f) for f in
             ("test_commsim.py", "test_scheduler.py", "test_mig.py", "test_simcore.py")]
    code = ("import sys\n"
            "from paper_2511_09143_b200.compat import install_migsim_alias\n"
            "install_migsim_alias()\n"
            "import pytest\n"
            f"sys.exit(pytest.main(['-q', '-p', 'no:cacheprovider', '--rootdir', {str(tmp_path)!r},"
            f" '-k', 'not ({OUT_OF_SCOPE})'] + {files!r}))\n")
    env = {**os.environ, "PYTHONDONTWRITEBYTECODE": "1", "PYTHONPATH": ROOT}
    r = subprocess.run([sys.executable, "-c", code], cwd=tmp_path, env=env,
                       capture_output=True, text=True, timeout=300)
    tail = r.stdout[-3000:]
    assert r.returncode == 0, tail
    passed = int(tail.strip().splitlines()[-1].split(" passed")[0].split()[-1])
    assert passed >= 72, tail
