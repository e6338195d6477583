"""Run the reference's OWN hot-path tests unmodified against the drop-in.

The tests are read from /root/reference/pkg/tests (never copied) with the
`mpsim` import shim (paper_2604_22228_b200/compat) first on the path, so
`from mpsim.paths import plan_paths` resolves to the B200 implementation.
Skipped where the reference tree is absent (e.g. on the GPU box).
"""

import os
import subprocess
import sys

import pytest

REF_TESTS = "/root/reference/pkg/tests"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COMPAT = os.path.join(ROOT, "paper_2604_22228_b200", "compat")

pytestmark = pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                                reason="reference tree not present")


@pytest.mark.parametrize("module", ["test_paths.py", "test_pipeline.py", "test_graph.py",
                                    "test_topology.py"])
def test_reference_module_passes_against_dropin(module, tmp_path):
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([COMPAT, ROOT]))
    res = subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
                          os.path.join(REF_TESTS, module), "--rootdir", str(tmp_path)],
                         cwd=tmp_path, env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout[-3000:] + res.stderr[-2000:]
    # the shim really served the drop-in, not the reference
    probe = subprocess.run([sys.executable, "-c", "import mpsim.paths as m; print(m.__file__)"],
                           cwd=tmp_path, env=env, capture_output=True, text=True)
    assert probe.stdout.strip().startswith(os.path.join(ROOT, "paper_2604_22228_b200"))
