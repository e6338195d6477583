"""CPU checks of bench.py's driver contract: the reference arm's JSON line
(keys, units, one line), that it never imports the product package, the
workload shape per world size, and the < 3 KB result line."""
import io
import json
import os
import subprocess
import sys
from contextlib import redirect_stdout

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import planner as op  # noqa: E402

MiB = 1 << 20


def _reference_line(*extra):
    code = (
        "import runpy, sys, json\n"
        f"sys.argv = ['bench.py', '--impl', 'reference', '--size', '{MiB + 12345}', '--window', '2',"
        " '--steps', '1', '--warmup', '1'" + "".join(f", {a!r}" for a in extra) + "]\n"
        f"runpy.run_path({os.path.join(ROOT, 'bench.py')!r}, run_name='__main__')\n"
        "bad = sorted(m for m in sys.modules if m.startswith('paper_2604_22228_b200'))\n"
        "print('PRODUCT_MODULES', json.dumps(bad))\n")
    env = dict(os.environ, WORLD_SIZE="1", RANK="0")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert lines[-1].startswith("PRODUCT_MODULES")
    return json.loads(lines[-2]), json.loads(lines[-1].split(" ", 1)[1])


def test_reference_arm_line_and_isolation():
    line, product = _reference_line()
    assert product == [], f"the reference arm imported the product: {product}"
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC
    assert line["unit"] == "GB/s" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["steps"] == 1 and line["warmup"] == 1 and line["n_gpus"] == 1
    cb = line["cpu_baseline"]
    assert cb["kind"] in ("port", "reference") and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert "workload" in line["config"] and line["config"]["msg_bytes"] == MiB + 12345


@pytest.mark.parametrize("world,shape", [(1, (1, True, 8)), (2, (1, True, 8)), (4, (3, True, 8)),
                                         (8, (7, True, 16))])
def test_plan_shape_follows_the_baseline_configs(world, shape):
    args = bench.argparse.Namespace(chunks=0)
    assert bench.plan_shape(args, world) == shape
    assert os.path.exists(bench.topo_file(world))


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_reference_plan_equals_the_oracle(world):
    """Both arms execute the reference planner's plan on the committed .topo."""
    args = bench.argparse.Namespace(chunks=0)
    g, host, k = bench.plan_shape(args, world)
    text = open(bench.topo_file(world)).read()
    kinds, chunks, _ = bench.reference_plan(text, world, g, host, 512 * MiB, k)
    t = op.parse_topology(text)
    paths = op.plan_paths(t, 0, 1, g, host)
    assert kinds == [p["kind"] for p in paths]
    assert [tuple(c) for c in chunks] == [tuple(c) for c in
                                           op.make_chunk_plan([p["share"] for p in paths], 512 * MiB, k)]
    assert sum(c[2] for c in chunks) == 512 * MiB


def test_emit_keeps_the_line_under_3kb():
    out = {"metric": "m", "value": 1.0, "notes": "x" * 4000, "multi_over_single": {str(i): i for i in range(50)}}
    buf = io.StringIO()
    with redirect_stdout(buf):
        bench.emit(out)
    line = buf.getvalue().strip()
    assert "\n" not in line and len(line) <= 3000
    assert json.loads(line)["value"] == 1.0


def test_host_rate_reads_the_planning_rate():
    assert bench.host_rate(open(bench.topo_file(1)).read()) == 1e9
