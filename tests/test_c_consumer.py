"""The C ABI from plain C: tests/c/plan_consumer.c (C99, gcc, no C++ or CUDA
headers) links libmpb200.so, plans GPU0 -> GPU1 and prints the chunk plan;
it must equal the oracle's plan (which is pinned to the reference's goldens)."""

import os
import shutil
import subprocess

import pytest

from oracle import planner as op
from paper_2604_22228_b200 import _lib, mesh_text

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "c", "plan_consumer.c")


@pytest.fixture(scope="module")
def consumer(tmp_path_factory):
    if not shutil.which("gcc"):
        pytest.skip("gcc not available")
    out = tmp_path_factory.mktemp("c") / "plan_consumer"
    libdir = os.path.dirname(_lib.LIB_PATH)
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-O2", "-I", os.path.join(ROOT, "include"),
                    SRC, "-o", str(out), "-L", libdir, "-l:libmpb200.so",
                    f"-Wl,-rpath,{libdir}"], check=True)
    return str(out)


@pytest.mark.parametrize("n,link,host,gpu_paths,use_host,chunks,size", [
    (2, 750e9, 55e9, 1, 1, 8, 64 << 20),
    (4, 900e9, 64e9, 3, 1, 8, 512 << 20),
    (8, 3.17e12, 6e9, 7, 1, 16, (512 << 20) + 12345),
    (8, 750e9, 55e9, 4, 0, 3, 30),
    (3, 2e12, 1e12, 2, 1, 1, 1)])
def test_c_consumer_plan_equals_oracle(consumer, tmp_path, n, link, host, gpu_paths, use_host,
                                       chunks, size):
    text = mesh_text("c", n, link, 1, 2e-6, host, 1e-5, "full")
    topo = tmp_path / "t.topo"
    topo.write_text(text)
    out = subprocess.run([consumer, str(topo), str(gpu_paths), str(use_host), str(chunks),
                          str(size)], capture_output=True, text=True, check=True).stdout
    lines = out.splitlines()
    shares = [float(l.split()[2]) for l in lines if l.startswith("share")]
    got = [tuple(int(x) for x in l.split()) for l in lines if not l.startswith("share")]
    t = op.parse_topology(text)
    opaths = op.plan_paths(t, 0, 1, gpu_paths, bool(use_host))
    assert shares == [p["share"] for p in opaths]
    assert got == [tuple(c) for c in op.make_chunk_plan([p["share"] for p in opaths], size, chunks)]
