"""Host-side pieces of the measured harness (no GPU): the Jacobi problem
spec mirrors bench.py:280-301 (validation messages and the halo formula,
test_bench.py:129-131), and result rows keep the reference's CSV layout."""

import pytest

from paper_2604_22228_b200 import PathConfig
from paper_2604_22228_b200 import measure as M

MiB = 1 << 20


def test_jacobi_halo_formula():
    spec = M.JacobiSpec(nx_values=[2 ** 27])
    assert spec.halo_bytes(2 ** 27) == 2 ** 27 * 8 // 4 == 256 * MiB
    assert M.JacobiSpec([1024], compute_time_per_cell=1e-9).compute_seconds(1024) == \
        1024 * 8 * 1e-9 / 4


@pytest.mark.parametrize("kw,msg", [({"ranks": 2}, "4 ranks"), ({"nx_values": []}, "no problem"),
                                    ({"nx_values": [6]}, "not divisible"),
                                    ({"element_size": 4}, "float64"), ({"timed": 0}, ">= 1")])
def test_jacobi_spec_validation(kw, msg):
    args = {"nx_values": [1024], **kw}
    with pytest.raises(ValueError, match=msg):
        M.JacobiSpec(**args)


def test_result_rows_and_speedup_lookup():
    spec = M.BenchmarkSpec("jacobi", [MiB], config=PathConfig(2, False, 4, graph_mode=True))
    res = M.BenchResult([M._row(spec, spec.config, MiB, "comm_time", 1e-3, 1.5),
                         M._row(spec, spec.config, MiB, "integrity", 1.0)])
    assert res.speedup(MiB, "comm_time") == 1.5 and res.integrity_all_clear
    with pytest.raises(KeyError, match="no speedup"):
        res.speedup(MiB, "integrity")
    assert res.to_csv().splitlines()[1] == "jacobi,b200,1048576,1,2,off,on,4,comm_time,0.001,1.5"


def test_host_rate_pick_prefers_the_smallest_within_tolerance():
    """The calibration curve is flat over a wide range of host rates; the
    pick is the smallest host rate within tolerance of the fastest run."""
    from paper_2604_22228_b200.tuner import pick_host_rate
    runs = [(1.000, 1e9, "t1", "ce"), (0.998, 4e9, "t4", "ce"), (0.996, 16e9, "t16", "ce"),
            (1.200, 55e9, "t55", "ce"), (0.999, 2e9, "t2", "sm")]
    assert pick_host_rate(runs, 0.005)[1] == 1e9
    assert pick_host_rate(runs, 0.0025)[1:3] == (4e9, "t4")
    assert pick_host_rate(runs, 0.0)[1] == 16e9
    assert pick_host_rate([(2.0, 8e9, "a", "sm")])[1] == 8e9
