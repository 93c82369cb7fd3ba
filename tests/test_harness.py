"""The reference's benchmark harness on the GPU path (bench.cpp:63-312)."""
import pytest


def test_setup_shapes_match_the_reference(ts):
    """make_setup / verify_setup / clamp_tb arithmetic (bench.cpp:104-107,
    192-226), incl. the golden row's 500x500 desk extent and tb=50
    (tests/golden/bench_row_golden.csv)."""
    from paper_2303_08365_b200 import harness as h
    spec = ts.find_benchmark("Heat-2D")
    assert h.make_setup(spec, "desk") == ([500, 500], [200, 200], 50)
    assert h.make_setup(ts.find_benchmark("Heat-3D"), "desk") == ([51, 51, 51], [20, 20, 20], 10)
    assert h.make_setup(ts.find_benchmark("Heat-1D"), "desk")[0] == [500000]
    assert h.verify_setup(ts.find_benchmark("Box-3D27P")) == ([24, 24, 24], [8, 8, 8], 3)
    assert h.clamp_tb(50, 200, 1) == 50 and h.clamp_tb(500, 8, 2) == 2


def test_csv_schema_extends_the_reference(ts):
    """The first 14 columns are the reference's CSV header (bench.cpp:289-292,
    tests/golden/bench_row_golden.csv)."""
    ref = ("name,path,dims,extent,T,tile,Tb,elapsed_s,stencils_per_s,verify,seed,"
           "ghost_recompute_points,mma_calls,messages")
    assert ts.csv_header().startswith(ref + ",")
    row = ts.run_benchmark("Heat-2D", path="vector")
    assert row["verify"] == "unsupported"
    assert ts.csv_row(row).split(",")[:2] == ["Heat-2D", "vector"]
    with pytest.raises(ValueError):
        ts.run_benchmark("Heat-2D", path="warp-drive")


@pytest.mark.gpu
@pytest.mark.parametrize("path", ["gpu", "tessellate", "naive"])
def test_benchmark_rows_verify_and_time(ts, path):
    """tests/python/test_smoke.py:136-140 on every GPU path, all 8 kernels."""
    for spec in ts.benchmark_table():
        row = ts.run_benchmark(spec.name, path=path, steps=4, seed=7)
        assert row["verify"] == "pass", row
        assert row["stencils_per_s"] > 0 and row["T"] == 4 and row["k"] >= 1


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["Heat-2D", "Heat-3D", "Box-3D27P"])
def test_hetero_path_rows_and_comm_log(ts, orc, ref, name, tmp_path):
    """--path hetero (bench.cpp:169-189) on two GPU slabs: the row verifies
    against the generic engine, its message count and ghost recompute are
    the reference run_heterogeneous's on the same grid and tile with the
    round length the GPU slabs use (tb clamped to the engine's fused depth:
    the deep halo is r*k planes), and the CLI writes the per-round CommLog
    CSV (scheduler.cpp:152-159)."""
    from paper_2303_08365_b200 import harness as h
    from paper_2303_08365_b200.cli import main
    import io
    spec = ts.find_benchmark(name)
    row = ts.run_benchmark(name, path="hetero", steps=7, seed=3)
    assert row["verify"] == "pass" and row["gpus"] == 2, row
    extent, tile, tb = h.make_setup(spec, "desk")
    g = ts.Grid(extent, [1] * len(extent))
    orc.fill_random(g, 3)
    assert 1 <= row["k"] <= tb
    msgs, ghost, _, _ = ref.run_heterogeneous(g, spec.kernel, 7, tile[0], row["k"])
    assert (row["messages"], row["ghost_recompute_points"]) == (msgs, ghost)
    csv = tmp_path / "rounds.csv"
    assert main(["run", "--name", name, "--path", "hetero", "--steps", "7",
                 "--comm-log", str(csv)], io.StringIO()) == 0
    lines = csv.read_text().splitlines()
    assert lines[0] == "round,direction,bytes,modeled_cost_alpha_beta,wall_seconds"
    assert len(lines) == 1 + msgs
