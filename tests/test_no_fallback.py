"""The product never routes through the oracle and has no CPU fallback:
importing the package loads no `oracle` module, no product source imports
it, and without the built CUDA library the package refuses to import."""
import os
import re
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2604_22228_b200")


def test_product_never_imports_the_oracle():
    code = ("import sys; import paper_2604_22228_b200 as mp; import paper_2604_22228_b200.engine, "
            "paper_2604_22228_b200.tuner, paper_2604_22228_b200.measure, paper_2604_22228_b200.group; "
            "print(sorted(m for m in sys.modules if m == 'oracle' or m.startswith('oracle.')))")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip().splitlines()[-1] == "[]"
    pat = re.compile(r"^\s*(from\s+oracle\b|import\s+oracle\b)", re.M)
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".c", ".cpp", ".cu", ".cuh", ".hpp")):
                text = open(os.path.join(dirpath, f), encoding="utf-8", errors="replace").read()
                assert not pat.search(text), f"{f} imports the oracle"


def test_package_refuses_to_import_without_the_cuda_library(tmp_path):
    dst = tmp_path / "paper_2604_22228_b200"
    shutil.copytree(PKG, dst, ignore=shutil.ignore_patterns("*.so", "_build", "__pycache__"))
    env = dict(os.environ, PYTHONPATH=str(tmp_path))
    out = subprocess.run([sys.executable, "-c", "import paper_2604_22228_b200"], cwd=str(tmp_path), env=env,
                         capture_output=True, text=True, timeout=300)
    assert out.returncode != 0, "imported without libmpb200.so: a silent fallback"
    assert "libmpb200" in (out.stderr + out.stdout)
