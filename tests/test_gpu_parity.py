"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden outputs and the pinned CPU oracle — bit for bit, every mode.

Tolerance: none. Every comparison is on the uint64/uint32 bit patterns
(the reference's grid_compare contract, grid.py:238-256); the FMA-free
W,E,S,C,N update makes the B200 schedules bitwise equal to jacobi_reference
for fp64, and to the fp32 restatement for fp32.
"""

import hashlib

import numpy as np
import pytest

from oracle import jacobi_c, jacobi_numpy
from paper_2306_03336_b200 import (DeviceModel, Grid2D, KernelConfig, Rect, StencilWeights, grid_extract,
                                   grid_new, j2d5pt, last_launch_count, plan_device_tiles, run_dtb,
                                   run_dtb_b200)
from paper_2306_03336_b200 import _native
from paper_2306_03336_b200.prng import random_interior

pytestmark = pytest.mark.gpu

W02 = StencilWeights.diffusive(0.2)
MIXED = StencilWeights(0.11, -0.2, 0.37, 0.5, -0.07)
# isotropic (w == e == s == n bitwise): the kernels' shared-product 6-op form
ISO_NEG = StencilWeights(-0.3, -0.3, -0.3, 0.7, -0.3)
# +0.0 / -0.0 weights: bitwise different, so NOT isotropic (x*0.0 and x*-0.0
# differ in sign); the all-+0.0 set is isotropic
ZERO_MIX = StencilWeights(0.0, -0.0, 0.0, 1.0, 0.0)
ZERO_ISO = StencilWeights(0.0, 0.0, 0.0, 1.0, 0.0)
WEIGHT_SETS = [MIXED, W02, ISO_NEG, ZERO_MIX, ZERO_ISO]
STREAM, NAIVE = _native.FLAG_FORCE_STREAM, _native.FLAG_FORCE_NAIVE
PIPE = _native.FLAG_FORCE_PIPE


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64 if a.dtype == np.float64 else np.uint32)


def same(a, b):
    return np.array_equal(bits(a), bits(b))


def rgrid(nx, ny, seed=0, ghost=0.0):
    return grid_new(nx, ny, random_interior(nx, ny, seed), ghost=ghost)


def test_kats_and_random_golden(golden):
    _, arr = golden
    steps = {"kat_spike1": 1, "kat_spike2": 2, "kat_drift": 1}
    for name in ["kat_spike1", "kat_spike2", "kat_fixed0.25", "kat_fixed0.125", "kat_drift"]:
        g = arr[f"{name}_in"]
        out = j2d5pt(Grid2D(g.shape[1] - 2, g.shape[0] - 2, g), arr[f"{name}_w"],
                     steps.get(name, 20))
        assert same(out.data, arr[f"{name}_out"]), name
    i = 0
    while f"rand{i}_in" in arr:
        g = arr[f"rand{i}_in"]
        grid = Grid2D(g.shape[1] - 2, g.shape[0] - 2, g)
        for flags in (0, STREAM, NAIVE):
            out, _ = run_dtb_b200(grid, arr[f"rand{i}_w"], int(arr[f"rand{i}_steps"]), flags=flags)
            assert same(out.data, arr[f"rand{i}_out"]), (i, flags)
        i += 1


def test_c1_matches_reference_hash(golden):
    meta, _ = golden
    for case in meta["cases"]:
        if not case["name"].startswith("C1"):
            continue
        g = rgrid(case["nx"], case["ny"], case["seed"], case["ghost"])
        for flags in (0, STREAM):
            out, _ = run_dtb_b200(g, case["weights"], case["steps"], flags=flags)
            assert sha(out.data) == case["sha256_out"], (case["name"], flags)
        assert last_launch_count() >= 1


def test_reference_batch_hashes(golden):
    meta, _ = golden
    for rec in meta["batch"]:
        g = rgrid(rec["nx"], rec["ny"], rec["seed"])
        out = j2d5pt(g, rec["weights"], rec["steps"])
        assert sha(out.data) == rec["sha256_out"], rec


def test_run_dtb_with_reference_plans(golden):
    meta, arr = golden
    for run in meta["runs"]:
        g = arr[f"{run['key']}_in"]
        grid = Grid2D(run["nx"], run["ny"], g)
        plan = plan_device_tiles((run["nx"], run["ny"]), DeviceModel("d", run["workers"], run["cap"]),
                                 run["t_depth"])
        v = Rect(*run["valid"]) if run["valid"] else None
        before = g.copy()
        out, rep = run_dtb(grid, W02, run["steps"], plan, KernelConfig(4), valid=v)
        assert same(out.data, arr[f"{run['key']}_out"]), run["key"]
        assert [rep.global_load_cells, rep.global_store_cells, rep.halo_exchanged_cells,
                rep.redundant_compute_cells, rep.useful_compute_cells,
                rep.scratchpad_peak_bytes, rep.elem_bytes] == run["report"]
        assert same(grid.data, before)  # input untouched


def test_pruned_valid_region_acceptance_2(golden):
    meta, _ = golden
    case = next(c for c in meta["cases"] if c["name"] == "pruned_560x536")
    g = rgrid(case["nx"], case["ny"], case["seed"])
    v = Rect(*case["valid"])
    for flags in (0, STREAM, NAIVE):
        out, _ = run_dtb_b200(g, case["weights"], case["steps"], valid=v, flags=flags)
        assert sha(grid_extract(out, v).data) == case["sha256_valid_out"], flags
        mask = np.ones((case["ny"], case["nx"]), bool)
        mask[v.y0:v.y1, v.x0:v.x1] = False
        assert same(out.interior[mask], g.interior[mask])


SHAPES = [(1, 1), (2, 2), (3, 7), (8, 8), (17, 5), (33, 29), (64, 64), (127, 130), (128, 126),
          (129, 64), (255, 257), (300, 41), (41, 300), (600, 500)]


@pytest.mark.parametrize("wi", range(len(WEIGHT_SETS)))
@pytest.mark.parametrize("nx,ny", SHAPES)
def test_modes_and_depths_match_oracle(nx, ny, wi):
    w = WEIGHT_SETS[wi]
    g = rgrid(nx, ny, nx * 1000 + ny, ghost=0.375)
    g.data[1:-1, 1:-1] -= 0.5  # both signs (signed-zero products for the zero weights)
    for steps in (1, 2, 5, 12):
        want = jacobi_c(g.data, w.astuple(), steps)
        for flags in (0, STREAM, NAIVE, PIPE):
            out, rep = run_dtb_b200(g, w, steps, flags=flags)
            assert same(out.data, want), (nx, ny, steps, flags)
            assert rep.useful_compute_cells == nx * ny * steps
        for depth in (2, 3, 6):
            out, _ = run_dtb_b200(g, w, steps, depth=depth)
            assert same(out.data, want), (nx, ny, steps, "depth", depth)
            out, _ = run_dtb_b200(g, w, steps, depth=depth, flags=STREAM)
            assert same(out.data, want), (nx, ny, steps, "stream depth", depth)


@pytest.mark.parametrize("nx,ny", [(5, 5), (64, 48), (300, 257), (1000, 200)])
def test_fp32_matches_fp32_oracle(nx, ny):
    g = rgrid(nx, ny, 77, ghost=0.5)
    for steps in (1, 4, 9):
        want = jacobi_numpy(g.data, W02.astuple(), steps, np.float32)
        for flags in (0, STREAM, NAIVE):
            out, _ = run_dtb_b200(g, W02, steps, flags=flags, dtype=np.float32)
            assert same(out.data.astype(np.float32), want), (nx, ny, steps, flags)


@pytest.mark.parametrize("nx,ny", [(129, 93), (300, 260), (700, 520)])
def test_poison_mode_does_not_leak(nx, ny):
    """NaN-poison debug mode (engine.py:16-20,174-177): every cell a correct
    schedule may no longer read is NaN-ed after each step; any stale read
    would surface as NaN in the result. Resident (forced), tile-streaming and
    default plans, several depths, multi-epoch runs."""
    g = rgrid(nx, ny, 7, ghost=1.5)
    want = jacobi_c(g.data, W02.astuple(), 16)
    for flags in (0, STREAM, _native.FLAG_FORCE_RESIDENT):
        for depth in (2, 4, 8):
            try:
                out, _ = run_dtb_b200(g, W02, 16, poison=True, flags=flags, depth=depth)
            except Exception as e:  # a forced resident plan may not fit this shape
                assert "fit" in str(e) or "feasible" in str(e), e
                continue
            assert not np.isnan(out.data).any(), (flags, depth)
            assert same(out.data, want), (flags, depth)


def test_determinism_and_input_untouched():
    g = rgrid(300, 300, 5)
    before = g.data.copy()
    a = j2d5pt(g, MIXED, 37)
    b = j2d5pt(g, MIXED, 37)
    assert same(a.data, b.data) and same(g.data, before)


def test_zero_steps_copy_and_negative_steps():
    g = rgrid(6, 5, 1, ghost=2.5)
    assert same(j2d5pt(g, W02, 0).data, g.data)
    with pytest.raises(ValueError):
        j2d5pt(g, W02, -1)


def test_c2_shape_resident_vs_oracle():
    # BASELINE config C2 geometry (1900^2 fp64, resident), 64 steps
    g = rgrid(1900, 1900, 1)
    out, rep = run_dtb_b200(g, W02, 64)
    assert same(out.data, jacobi_c(g.data, W02.astuple(), 64))
    assert rep.scratchpad_peak_bytes <= 232448


@pytest.mark.slow
def test_c2_full_10000_steps_bitwise():
    # the headline configuration, all 10^4 steps, against the C oracle
    g = rgrid(1900, 1900, 1)
    out, _ = run_dtb_b200(g, W02, 10000)
    assert same(out.data, jacobi_c(g.data, W02.astuple(), 10000))


def test_c3a_shape_fp32_resident_vs_oracle():
    g = rgrid(2700, 2700, 1)
    out, _ = run_dtb_b200(g, W02, 40, dtype=np.float32)
    assert same(out.data.astype(np.float32), jacobi_c(g.data, W02.astuple(), 40, np.float32))


def test_streaming_large_fp64_vs_oracle():
    g = rgrid(4096, 3000, 3)
    out, _ = run_dtb_b200(g, MIXED, 24)
    assert same(out.data, jacobi_c(g.data, MIXED.astuple(), 24))


def test_streaming_c3b_shape_fp32_vs_oracle():
    g = rgrid(8192, 8192, 1)
    out, _ = run_dtb_b200(g, W02, 12, dtype=np.float32)
    assert same(out.data.astype(np.float32), jacobi_c(g.data, W02.astuple(), 12, np.float32))


def test_device_tensor_entry_and_gpu_fill():
    import torch
    from paper_2306_03336_b200 import j2d5pt_device
    from paper_2306_03336_b200.prng import fill_random_device
    nx, ny = 777, 555
    a = torch.empty((ny + 2, nx + 2), dtype=torch.float64, device="cuda")
    b = torch.empty_like(a)
    fill_random_device(a, nx, ny, 42, ghost=0.25)
    host = rgrid(nx, ny, 42, ghost=0.25)
    assert same(a.cpu().numpy(), host.data)
    j2d5pt_device(a, b, nx, ny, MIXED, 33)
    torch.cuda.synchronize()
    assert same(b.cpu().numpy(), jacobi_c(host.data, MIXED.astuple(), 33))


@pytest.mark.parametrize("w", [MIXED, W02])
@pytest.mark.parametrize("nx,ny", [(1, 1), (3, 7), (9, 7), (64, 48), (129, 64), (300, 257),
                                   (1000, 37), (600, 2000)])
def test_pipe_kernel_matches_oracle(nx, ny, w):
    g = rgrid(nx, ny, nx * 7 + ny, ghost=0.375)
    for steps in (1, 2, 3, 7, 8, 9, 17):
        want = jacobi_c(g.data, w.astuple(), steps)
        out, _ = run_dtb_b200(g, w, steps, flags=PIPE)
        assert same(out.data, want), (nx, ny, steps)


def test_pipe_kernel_fp32_and_large():
    g = rgrid(4000, 3000, 5)
    out, _ = run_dtb_b200(g, W02, 24, flags=PIPE)
    assert same(out.data, jacobi_c(g.data, W02.astuple(), 24))
    out, _ = run_dtb_b200(g, W02, 16, flags=PIPE, dtype=np.float32)
    assert same(out.data.astype(np.float32), jacobi_c(g.data, W02.astuple(), 16, np.float32))


def _device_bitwise_vs_naive(nx, ny, steps, dtype, seed=1):
    """Full-size check without a CPU oracle: the chosen schedule and the naive
    one-step-per-launch kernel (an independent code path) on device buffers."""
    import torch
    from paper_2306_03336_b200 import j2d5pt_device
    from paper_2306_03336_b200.prng import fill_random_device
    tdt = torch.float64 if dtype == "f64" else torch.float32
    pitch = (nx + 2 + 31) // 32 * 32
    a = torch.empty((ny + 2, pitch), dtype=tdt, device="cuda")
    fill_random_device(a, nx, ny, seed, ghost=0.125)
    b = torch.empty_like(a)
    c = torch.empty_like(a)
    j2d5pt_device(a, b, nx, ny, MIXED, steps)
    j2d5pt_device(a, c, nx, ny, MIXED, steps, flags=_native.FLAG_FORCE_NAIVE)
    torch.cuda.synchronize()
    ib = torch.int64 if dtype == "f64" else torch.int32
    eq = torch.equal(b[:, :nx + 2].view(ib), c[:, :nx + 2].view(ib))
    del a, b, c
    torch.cuda.empty_cache()
    return eq


def test_c4_full_size_vs_naive():
    # BASELINE config C4 geometry (16384^2 fp64, pipe), two full 8-step passes
    assert _device_bitwise_vs_naive(16384, 16384, 16, "f64")


def test_c5_full_domain_single_gpu_vs_naive():
    # BASELINE config C5's whole 32768^2 fp64 domain on one B200 (8.6 GB per buffer)
    assert _device_bitwise_vs_naive(32768, 32768, 9, "f64", seed=5)


def test_c3b_full_size_fp32_vs_naive():
    assert _device_bitwise_vs_naive(8192, 8192, 20, "f32", seed=2)


def test_randomized_shapes_every_mode():
    """Fuzz across the planner's mode boundaries (resident / pipe / tile
    streaming / forced depths), odd sizes, both dtypes, mixed-sign weights."""
    rng = np.random.default_rng(20261018)
    PIPE_, RES = _native.FLAG_FORCE_PIPE, _native.FLAG_FORCE_RESIDENT
    for case in range(28):
        nx = int(rng.integers(1, 700))
        ny = int(rng.integers(1, 700))
        steps = int(rng.integers(1, 40))
        dt = np.float32 if case % 3 == 2 else np.float64
        g = rgrid(nx, ny, 1000 + case, ghost=float(rng.choice([0.0, 0.375, -1.5])))
        w = StencilWeights(*(float(x) for x in rng.uniform(-0.6, 0.6, 5)))
        want = jacobi_c(g.data, w.astuple(), steps, dt)
        for flags, depth in ((0, None), (STREAM, None), (PIPE_, None), (RES, None),
                             (0, int(rng.integers(1, 9)))):
            if depth is not None and steps % depth:
                continue
            try:
                out, _ = run_dtb_b200(g, w, steps, dtype=dt, flags=flags, depth=depth)
            except Exception as e:  # a forced mode may not fit this shape
                assert "fit" in str(e) or "feasible" in str(e) or "resident" in str(e), e
                continue
            assert same(out.data.astype(dt), want), (nx, ny, steps, dt, flags, depth)


_KNOB_SCRIPT = r"""
import sys
sys.path[:0] = ['.', 'tests']
from test_gpu_parity import _device_bitwise_vs_naive
from paper_2306_03336_b200.planner import plan_b200
for nx, ny, dt in ((1900, 1900, 'f64'), (2700, 2700, 'f32'), (700, 900, 'f64'), (1300, 600, 'f32')):
    p = plan_b200(nx, ny, 8 if dt == 'f64' else 4, 12, 1)
    ok = _device_bitwise_vs_naive(nx, ny, 12, dt, seed=nx)
    print(nx, ny, dt, p.mode, p.warps, p.tiles_x * p.tiles_y, p.ctas, ok)
"""


@pytest.mark.parametrize("env", ["DTB_MAX_TILES=37", "DTB_MAX_TILES=90"])
def test_planner_experiment_knobs_stay_bitwise(env):
    """The planner's tile-count cap selects other resident tilings (or pushes
    resident shapes into the pipe); each must still be bitwise equal to the
    naive kernel."""
    import os
    import subprocess
    import sys
    key, val = env.split("=")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _KNOB_SCRIPT], cwd=root, capture_output=True,
                       text=True, env={**os.environ, key: val}, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.strip().splitlines()
    assert len(lines) == 4 and all(l.endswith("True") for l in lines), r.stdout
    assert all(int(l.split()[5]) <= int(val) for l in lines if l.split()[3] == "0"), r.stdout


def test_misaligned_origins_valid_windows_and_offset_views():
    """Odd-column valid windows (fp64) and x0 % 4 != 0 (fp32) put the solved
    grid's origin off a 16-byte boundary; the device entry takes offset views
    too. All must be bitwise equal to the oracle (the solve stages through an
    aligned copy)."""
    import torch
    from paper_2306_03336_b200 import grid_extract, j2d5pt_device
    w = MIXED
    g = rgrid(300, 260, 3, ghost=0.125)
    for v, dt in ((Rect(17, 9, 250, 231), np.float64), (Rect(1, 1, 7, 5), np.float64),
                  (Rect(5, 3, 201, 100), np.float32), (Rect(2, 0, 298, 260), np.float32)):
        for flags in (0, STREAM, _native.FLAG_FORCE_PIPE):
            try:
                out, _ = run_dtb_b200(g, w, 24, valid=v, dtype=dt, flags=flags)
            except Exception as e:
                assert "fit" in str(e) or "feasible" in str(e), e
                continue
            sub = grid_extract(g, v)
            want = jacobi_c(sub.data, w.astuple(), 24, dt)
            got = out.data[v.y0:v.y0 + v.height + 2, v.x0:v.x0 + v.width + 2]
            assert same(got.astype(dt), want), (v, dt, flags)
    # a device view starting one column into a buffer
    nx, ny = 129, 77
    base = torch.zeros((ny + 2, 1 + 160), dtype=torch.float64, device="cuda")
    gg = rgrid(nx, ny, 9, ghost=0.5)
    base[:, 1:nx + 3] = torch.from_numpy(gg.data).cuda()
    src = base[:, 1:]
    dst = torch.zeros_like(base)[:, 1:]
    j2d5pt_device(src, dst, nx, ny, w, 10)
    want = jacobi_c(gg.data, w.astuple(), 10)
    assert np.array_equal(dst[:, :nx + 2].cpu().numpy().view(np.uint64), want.view(np.uint64))


def test_fuzz_every_entry_point():
    """tools/fuzz.py: random shapes, odd-column valid windows, forced modes and
    depths, n_gpus slabs (fused / copy), offset device views — all bitwise
    against the C oracle (3,900 cases at seeds 1-3 on the round-1 box)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, os.path.join(root, "tools", "fuzz.py"), "300", "11"],
                       cwd=root, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_device_buffers_of_other_dtypes_are_rejected():
    import torch
    from paper_2306_03336_b200 import j2d5pt_device
    from paper_2306_03336_b200.prng import fill_random_device, fill_random_rows_device
    a = torch.zeros((18, 32), dtype=torch.float16, device="cuda")
    with pytest.raises(ValueError, match="dtype"):
        j2d5pt_device(a, a.clone(), 16, 16, W02, 2)
    with pytest.raises(ValueError, match="dtype"):
        fill_random_device(a, 16, 16, 1)
    with pytest.raises(ValueError, match="dtype"):
        fill_random_rows_device(a, 16, 16, 1, 0)
    with pytest.raises(ValueError, match="dtype"):
        fill_random_rows_device(a.float(), 16, 16, 1, 0)  # the row fill is fp64 only


def test_offset_view_with_valid_window_leaves_outside_columns_untouched():
    """with valid=, the frozen cells are copied with a 2-D copy of
    the view's nx+2 columns only; the columns of the allocation outside the
    view keep their sentinels (and an offset view reads nothing past its end)."""
    import torch
    from paper_2306_03336_b200 import j2d5pt_device
    nx, ny, steps = 129, 77, 10
    v = Rect(13, 5, 100, 60)
    gg = rgrid(nx, ny, 11, ghost=0.5)
    sentinel = -12345.5
    base_in = torch.full((ny + 2, 1 + 160), sentinel, dtype=torch.float64, device="cuda")
    base_in[:, 1:nx + 3] = torch.from_numpy(gg.data).cuda()
    base_out = torch.full_like(base_in, sentinel)
    j2d5pt_device(base_in[:, 1:], base_out[:, 1:], nx, ny, MIXED, steps, valid=v)
    out = base_out.cpu().numpy()
    assert (out[:, 0] == sentinel).all() and (out[:, nx + 3:] == sentinel).all()
    sub = grid_extract(gg, v)
    want = jacobi_c(sub.data, MIXED.astuple(), steps)
    got = out[:, 1:nx + 3][v.y0:v.y0 + v.height + 2, v.x0:v.x0 + v.width + 2]
    assert same(got, want)
    # cells outside the valid window are carried over unchanged
    full = out[:, 1:nx + 3].copy()
    mask = np.ones_like(full, dtype=bool)
    mask[v.y0 + 1:v.y0 + v.height + 1, v.x0 + 1:v.x0 + v.width + 1] = False
    assert np.array_equal(full[mask].view(np.uint64), gg.data[mask].view(np.uint64))


def test_device_entry_rejects_buffers_on_two_devices():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    from paper_2306_03336_b200 import j2d5pt_device
    a = torch.zeros((18, 32), dtype=torch.float64, device="cuda:0")
    b = torch.zeros((18, 32), dtype=torch.float64, device="cuda:1")
    with pytest.raises(ValueError, match="cuda:1"):
        j2d5pt_device(a, b, 16, 16, W02, 2)
