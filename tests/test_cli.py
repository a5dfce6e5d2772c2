"""The dtb-stencil front end (paper_2306_03336_b200/cli.py), mirroring the
reference's tests/test_cli.py: exit codes, CSV schema, plan JSON, presets,
fixture chaining. Solves run on the GPU (marked); usage/plan/preset paths
need none."""

import json

import numpy as np
import pytest

import paper_2306_03336_b200.cli as cli
from paper_2306_03336_b200.grid import (grid_compare, grid_from_bytes, grid_new, grid_to_bytes,
                                        load_grid, save_grid)
from paper_2306_03336_b200.metrics import RUN_CSV_COLUMNS, run_csv_row
from paper_2306_03336_b200.prng import random_interior

COL = RUN_CSV_COLUMNS.index


def run_cli(capsys, *argv):
    code = cli.main(list(argv))
    cap = capsys.readouterr()
    return code, cap.out, cap.err


# --- CPU: usage, plan, presets, fixtures ---------------------------------------

@pytest.mark.parametrize("argv", [
    ("verify", "--nx", "8", "--ny", "8", "--t", "2", "--steps", "5"),
    ("verify", "--nx", "8", "--ny", "8", "--t", "0"),
    ("verify", "--ny", "8", "--t", "1"),
    ("verify", "--nx", "8", "--ny", "8", "--device", "nope"),
    ("verify", "--nx", "8", "--ny", "8", "--device", "b200", "--workers", "2",
     "--capacity", "100"),
    ("verify", "--nx", "8", "--ny", "8", "--workers", "2"),
    ("verify", "--nx", "8", "--ny", "8", "--ilp", "0"),
    ("verify", "--nx", "8", "--ny", "8", "--threads", "0"),
    ("verify", "--nx", "8", "--ny", "8", "--pruned", "16x4"),
    ("verify", "--nx", "8", "--ny", "8", "--alpha", "0.1", "--weights", "1,0,0,0,0"),
    ("verify", "--nx", "8", "--ny", "8", "--weights", "1,2,3"),
    ("run", "--nx", "8"),
    ("sweep", "--t-list", ""),
    ("sweep", "--sizes", "0x4"),
    ("nonsense",),
])
def test_usage_errors_exit_64(capsys, argv):
    assert run_cli(capsys, *argv)[0] == 64


def test_help_exits_zero(capsys):
    code, out, _ = run_cli(capsys, "--help")
    assert code == 0 and "verify" in out and "sweep" in out


def test_plan_prints_reference_json(capsys):
    # the reference's golden plan (test_cli.py:174-187)
    code, out, _ = run_cli(capsys, "plan", "--nx", "16", "--ny", "16", "--t", "1",
                           "--workers", "2", "--capacity", "2048")
    assert code == 0
    plan = json.loads(out)
    assert plan["domain"] == {"nx": 16, "ny": 16}
    assert plan["t_depth"] == 1 and plan["footprint_bytes"] == 1936
    assert plan["device"]["workers"] == 2 and len(plan["tiles"]) == 2
    tile = plan["tiles"][0]
    assert tile["interior"] == {"x0": 0, "y0": 0, "width": 16, "height": 9}
    assert tile["halo"] == 1
    assert [s["owner"] for s in tile["subtiles"]] == [0, 1]


def test_plan_infeasible_exits_two(capsys):
    code, _, err = run_cli(capsys, "plan", "--nx", "4", "--ny", "4", "--t", "2",
                           "--workers", "1", "--capacity", "64")
    assert code == 2 and "560" in err


def test_plan_native_is_the_b200_schedule(capsys):
    code, out, _ = run_cli(capsys, "plan", "--nx", "1900", "--ny", "1900", "--t", "4",
                           "--native")
    assert code == 0
    p = json.loads(out)
    assert p["mode"] == "resident" and p["halo"] == 4 and p["ctas"] <= 148


def test_presets_and_footprints(capsys, tmp_path):
    code, out, _ = run_cli(capsys, "presets")
    assert code == 0
    assert out.splitlines()[0] == "name,workers,scratchpad_bytes_per_worker,total_bytes,total"
    assert "b200,148,232448,34402304,32.81 MB" in out
    p = tmp_path / "toy.ini"
    p.write_text("[toy]\nworkers = 2\nscratchpad_bytes_per_worker = 4096\n")
    code, out, _ = run_cli(capsys, "presets", "--presets", str(p))
    assert out.splitlines()[1] == "toy,2,4096,8192,8 KB"
    code, out, _ = run_cli(capsys, "footprints", "--device", "b200")
    assert out == "name,scratchpad\nStencilGen,4.32 MB\nAN5D,0.864 MB\ndtb-b200,32.81 MB\n"


def test_fixture_roundtrip(tmp_path):
    g = grid_new(7, 5, random_interior(7, 5, 3), ghost=0.125)
    g.data[0, 3] = -0.0
    blob = grid_to_bytes(g)
    assert len(blob) == 16 + 9 * 7 * 8
    assert grid_compare(grid_from_bytes(blob), g).bit_equal
    path = tmp_path / "g.grid"
    save_grid(g, path)
    h = load_grid(path)
    assert np.array_equal(h.data.view(np.uint64), g.data.view(np.uint64))
    with pytest.raises(ValueError):
        grid_from_bytes(blob[:-8])
    with pytest.raises(ValueError):
        grid_from_bytes(b"\x00" * 4)


def test_csv_row_schema():
    assert len(RUN_CSV_COLUMNS) == 35
    row = run_csv_row({"status": "ok", "nx": 3, "bit_equal": True})
    cells = row.split(",")
    assert len(cells) == 35 and cells[COL("bit_equal")] == "true" and cells[COL("seed")] == ""
    with pytest.raises(ValueError):
        run_csv_row({"bogus": 1})


# --- GPU: solves through the B200 kernels --------------------------------------

RUN_ARGS = ("run", "--nx", "40", "--ny", "36", "--t", "2", "--steps", "6",
            "--workers", "2", "--capacity", "8192")


@pytest.mark.gpu
def test_verify_bitwise(capsys):
    code, out, _ = run_cli(capsys, "verify", "--nx", "96", "--ny", "80", "--t", "4",
                           "--steps", "12", "--seed", "7")
    assert code == 0 and "bit_equal=true" in out and "max_abs_diff=0.0" in out


@pytest.mark.gpu
def test_verify_pruned_and_fp32(capsys):
    code, out, _ = run_cli(capsys, "verify", "--nx", "24", "--ny", "20", "--pruned", "16x12",
                           "--t", "2", "--steps", "6", "--workers", "2", "--capacity", "8192")
    assert code == 0 and "bit_equal=true" in out
    code, out, _ = run_cli(capsys, "verify", "--nx", "64", "--ny", "48", "--t", "4",
                           "--steps", "8", "--dtype", "f32")
    assert code == 0 and "bit_equal=true" in out


@pytest.mark.gpu
def test_verify_mismatch_exits_one(capsys, monkeypatch):
    real = cli.run_dtb

    def skewed(*a, **k):
        out, rep = real(*a, **k)
        out.interior[0, 0] += 1.0
        return out, rep

    monkeypatch.setattr(cli, "run_dtb", skewed)
    code, out, _ = run_cli(capsys, "verify", "--nx", "6", "--ny", "6", "--t", "1")
    assert code == 1 and "bit_equal=false" in out and "first_mismatch=0,0" in out


@pytest.mark.gpu
def test_run_emits_csv_row_and_is_reproducible(capsys):
    code, out, _ = run_cli(capsys, *RUN_ARGS, "--check")
    assert code == 0
    header, row = out.strip().split("\n")
    assert header == ",".join(RUN_CSV_COLUMNS)
    cells = row.split(",")
    assert cells[COL("status")] == "ok" and cells[COL("device")] == "custom"
    assert cells[COL("bit_equal")] == "true" and int(cells[COL("tiles")]) >= 1
    assert float(cells[COL("wall_time_s")]) > 0
    _, out2, _ = run_cli(capsys, *RUN_ARGS, "--check", "--no-header")
    a, b = row.split(","), out2.strip().split(",")
    timing = {COL("wall_time_s"), COL("host_model_gflops")}
    assert all(x == y for i, (x, y) in enumerate(zip(a, b)) if i not in timing)
    code, out, _ = run_cli(capsys, *RUN_ARGS, "--format", "json")
    rec = json.loads(out)
    assert rec["status"] == "ok" and rec["useful_compute_cells"] == 40 * 36 * 6


@pytest.mark.gpu
def test_run_save_and_load_grid_chain(capsys, tmp_path):
    from paper_2306_03336_b200 import StencilWeights, j2d5pt
    p1, p2 = str(tmp_path / "a.grid"), str(tmp_path / "b.grid")
    args = ("--t", "1", "--steps", "2", "--no-header")
    assert run_cli(capsys, "run", "--nx", "8", "--ny", "8", *args, "--save-grid", p1)[0] == 0
    code, out, _ = run_cli(capsys, "run", "--load-grid", p1, *args, "--save-grid", p2)
    assert code == 0 and out.split(",")[COL("seed")] == ""
    start = grid_new(8, 8, random_interior(8, 8, 1))
    want = j2d5pt(start, StencilWeights.diffusive(0.2), 4)
    assert grid_compare(load_grid(p2), want).bit_equal
    assert run_cli(capsys, "run", "--load-grid", p1, "--nx", "9", *args)[0] == 64


@pytest.mark.gpu
def test_sweep_rows_and_infeasible(capsys, tmp_path):
    p = tmp_path / "c.ini"
    p.write_text("[toy]\nworkers = 2\nscratchpad_bytes_per_worker = 4096\n"
                 "[nano]\nworkers = 1\nscratchpad_bytes_per_worker = 600\n")
    code, out, _ = run_cli(capsys, "sweep", "--presets", str(p), "--devices", "toy,nano",
                           "--sizes", "16x16,12x8", "--t-list", "1,4", "--check")
    assert code == 0
    rows = [r.split(",") for r in out.strip().split("\n")[1:]]
    assert len(rows) == 8
    status = [(r[COL("device")], r[COL("t_depth")], r[COL("status")]) for r in rows]
    assert ("nano", "4", "infeasible") in status
    assert all(r[COL("bit_equal")] == "true" for r in rows if r[COL("status")] == "ok")
