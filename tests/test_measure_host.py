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
