"""Measured harness in the reference's CSV schema (bench.py:33): rows parse
with the reference's own column layout and carry real, positive values."""

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_bw_bibw_latency_rows():
    from paper_2604_22228_b200 import Engine, PathConfig
    from paper_2604_22228_b200 import measure as M
    eng = Engine.loopback(2)
    cfg = PathConfig(num_gpu_paths=1, host_path_enabled=True, max_chunks=4, graph_mode=True)
    sizes = [1 << 20, 8 << 20]
    bw = M.run_bw(M.BenchmarkSpec("omb_bw", sizes, window=4, iterations=3, config=cfg), eng)
    bibw = M.run_bibw(M.BenchmarkSpec("omb_bibw", sizes, window=2, iterations=2, config=cfg), eng)
    lat = M.run_latency(M.BenchmarkSpec("omb_latency", sizes, iterations=3, config=cfg), eng)
    for res in (bw, bibw, lat):
        lines = res.to_csv().splitlines()
        assert lines[0] == M.CSV_HEADER
        for line in lines[1:]:
            f = line.split(",")
            assert len(f) == 11 and float(f[9]) >= 0.0
    assert bw.value(8 << 20, "bandwidth") > 1e9
    assert bibw.value(8 << 20, "bandwidth") > 1e9
    assert lat.value(1 << 20, "phase_instantiation_first") > 0.0
    import paper_2604_22228_b200 as mp
    topo = eng.topology
    plan = mp.make_chunk_plan(mp.plan_paths(topo, topo.device(0), topo.device(1), cfg), 1 << 20, 4)
    assert lat.value(1 << 20, "nodes") == mp.build_graph(plan).node_count
    eng.close()


@pytest.mark.parametrize("window", [1, 16, 64])
def test_program_window_is_exact(window):
    """A window posted as one send_many program over W distinct pairs: every
    pair byte-exact (run_bw checks), odd and tiny sizes included."""
    from paper_2604_22228_b200 import Engine, PathConfig
    from paper_2604_22228_b200 import measure as M
    eng = Engine.loopback(2)
    sizes = [1, 4096 + 3, 65536, (1 << 20) + 12345]
    res = M.run_bw(M.BenchmarkSpec("omb_bw_program", sizes, window=window, iterations=2,
                                   warmup=1, config=PathConfig(1, False, 1, True)), eng,
                   program=True)
    assert res.value(65536, "bandwidth") > 0.0
    with pytest.raises(ValueError):
        M.run_bw(M.BenchmarkSpec("omb_bw_program", [4096], window=65), eng, program=True)
    eng.close()


def test_jacobi_ring_exchange_is_exact_and_timed():
    from paper_2604_22228_b200 import Engine, PathConfig
    from paper_2604_22228_b200 import measure as M
    eng = Engine.loopback(4)
    nx = 1 << 20                                   # 2 MiB halo per neighbour
    spec = M.JacobiSpec(nx_values=[nx], iterations=100, timed=4)
    for cfg in (PathConfig(2, False, 4, graph_mode=True), PathConfig(1, True, 2),
                PathConfig(3, True, 8, graph_mode=True)):
        res = M.run_jacobi(spec, cfg, eng)
        halo = spec.halo_bytes(nx)
        assert res.integrity_all_clear and res.value(halo, "integrity") == 1.0
        assert res.value(halo, "comm_time") > 0 and res.speedup(halo, "comm_time") > 0
        assert res.value(halo, "runtime") == res.value(halo, "comm_time")  # no compute
    modeled = M.JacobiSpec(nx_values=[nx], iterations=100, timed=4, compute_time_per_cell=1e-9)
    res = M.run_jacobi(modeled, PathConfig(2, False, 4, graph_mode=True), eng, compute="kernel")
    halo = modeled.halo_bytes(nx)
    assert res.value(halo, "runtime") > res.value(halo, "comm_time") + 100 * \
        modeled.compute_seconds(nx)
    assert res.integrity_all_clear
    assert len(res.to_csv().splitlines()) == 4
    eng.close()


def test_jacobi_needs_four_ranks():
    from paper_2604_22228_b200 import Engine, PathConfig
    from paper_2604_22228_b200 import measure as M
    eng = Engine.loopback(2)
    with pytest.raises(ValueError, match="4-accelerator"):
        M.run_jacobi(M.JacobiSpec(nx_values=[1 << 20]), PathConfig(), eng)
    eng.close()
