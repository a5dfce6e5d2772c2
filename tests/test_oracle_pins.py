"""Pin the CPU oracle (oracle/) to the reference's own outputs.

The fixtures in tests/golden were produced by importing the reference package
(tests/golden/make_golden.py). Both restatements — numpy and plain C — must
reproduce them bit for bit before anything is checked against them.
"""

import hashlib

import numpy as np
import pytest

from oracle import jacobi_c, jacobi_numpy, random_interior_c
from paper_2306_03336_b200.grid import grid_new
from paper_2306_03336_b200.prng import random_interior, splitmix64


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


KATS = ["kat_spike1", "kat_spike2", "kat_fixed0.25", "kat_fixed0.125", "kat_drift"]


@pytest.mark.parametrize("name", KATS)
@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_oracle_reproduces_reference_kats(golden, name, impl):
    _, arr = golden
    steps = {"kat_spike1": 1, "kat_spike2": 2, "kat_drift": 1}.get(name, 20)
    fn = jacobi_numpy if impl == "numpy" else jacobi_c
    out = fn(arr[f"{name}_in"], arr[f"{name}_w"], steps)
    assert np.array_equal(bits(out), bits(arr[f"{name}_out"]))


def test_spike_two_steps_closed_form(golden):
    # test_oracle.py:40-53: center = v+v+v+v+v, ring = v+v with v = 0.2*0.2
    _, arr = golden
    out = jacobi_c(arr["kat_spike2_in"], arr["kat_spike2_w"], 2)
    v = 0.2 * 0.2
    assert out[2, 2] == v + v + v + v + v and out[1, 2] == v + v


@pytest.mark.parametrize("impl", ["numpy", "c"])
def test_oracle_reproduces_reference_random_grids(golden, impl):
    _, arr = golden
    fn = jacobi_numpy if impl == "numpy" else jacobi_c
    i = 0
    while f"rand{i}_in" in arr:
        out = fn(arr[f"rand{i}_in"], arr[f"rand{i}_w"], int(arr[f"rand{i}_steps"]))
        assert np.array_equal(bits(out), bits(arr[f"rand{i}_out"])), f"rand{i}"
        i += 1
    assert i >= 10


def test_c_oracle_reproduces_reference_c1(golden):
    meta, _ = golden
    for case in meta["cases"]:
        if not case["name"].startswith("C1"):
            continue
        g = grid_new(case["nx"], case["ny"], random_interior(case["nx"], case["ny"], case["seed"]),
                     ghost=case["ghost"])
        out = jacobi_c(g.data, case["weights"], case["steps"])
        assert sha(out) == case["sha256_out"], case["name"]
        for key, v in case.get("samples", {}).items():
            x, y = map(int, key.split(","))
            assert out[y + 1, x + 1] == v


def test_c_oracle_reproduces_reference_batch(golden):
    meta, _ = golden
    for rec in meta["batch"]:
        g = grid_new(rec["nx"], rec["ny"], random_interior(rec["nx"], rec["ny"], rec["seed"]))
        out = jacobi_c(g.data, rec["weights"], rec["steps"], threads=4)
        assert sha(out) == rec["sha256_out"], rec


def test_c_oracle_reproduces_reference_pruned_case(golden):
    meta, _ = golden
    case = next(c for c in meta["cases"] if c["name"] == "pruned_560x536")
    g = grid_new(case["nx"], case["ny"], random_interior(case["nx"], case["ny"], case["seed"]))
    x0, y0, w, h = case["valid"]
    sub = g.data[y0:y0 + h + 2, x0:x0 + w + 2]
    assert sha(jacobi_c(sub, case["weights"], case["steps"])) == case["sha256_valid_out"]


def test_c_oracle_thread_count_independent():
    g = grid_new(61, 47, random_interior(61, 47, 3), ghost=0.25)
    w = (0.11, -0.2, 0.37, 0.5, -0.07)
    ref = jacobi_c(g.data, w, 9, threads=1)
    for t in (2, 3, 8, 64):
        assert np.array_equal(bits(jacobi_c(g.data, w, 9, threads=t)), bits(ref))


def test_fp32_oracles_agree():
    g = grid_new(45, 38, random_interior(45, 38, 8), ghost=0.5)
    w = (0.2, 0.2, 0.2, 0.19999999999999996, 0.2)
    a = jacobi_numpy(g.data, w, 11, np.float32)
    b = jacobi_c(g.data, w, 11, np.float32)
    assert a.dtype == np.float32 and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_zero_steps_is_a_copy():
    g = grid_new(5, 4, random_interior(5, 4, 9), ghost=2.5)
    assert np.array_equal(bits(jacobi_c(g.data, (0.2,) * 5, 0)), bits(g.data))


def test_prng_frozen_vectors(golden):
    meta, _ = golden
    assert [int(v) for v in splitmix64(1234567, 5)] == meta["prng"]["splitmix64_1234567"]
    assert random_interior(3, 2, 9).tolist() == meta["prng"]["random_interior_3x2_seed9"]
    assert np.array_equal(random_interior_c(30, 20, 77), random_interior(30, 20, 77))


def test_reference_structured_ports_reproduce_reference_runs(golden):
    """oracle/engine_port.py (the bench's BASELINE.md §4 CPU legs): the
    row-wise jacobi_reference restatement and the DTB engine restatement
    reproduce the reference's run_dtb outputs (tests/golden, no valid region)
    and the C oracle, bit for bit."""
    from oracle.engine_port import jacobi_rowwise, run_dtb_port
    from paper_2306_03336_b200 import DeviceModel, StencilWeights, plan_device_tiles
    meta, arr = golden
    w = StencilWeights.diffusive(0.2).astuple()
    checked = 0
    for r in meta["runs"]:
        if r["valid"] is not None:
            continue
        g = arr[f"{r['key']}_in"]
        want = arr[f"{r['key']}_out"]
        plan = plan_device_tiles((r["nx"], r["ny"]), DeviceModel("d", r["workers"], r["cap"]),
                                 r["t_depth"])
        for threads in (1, 3):
            assert np.array_equal(bits(run_dtb_port(g, w, r["steps"], plan, threads)),
                                  bits(want)), (r["key"], threads)
        assert np.array_equal(bits(jacobi_rowwise(g, w, r["steps"])), bits(want)), r["key"]
        checked += 1
    assert checked >= 5
    g = grid_new(67, 45, random_interior(67, 45, 3), ghost=0.5).data
    mixed = (0.11, -0.2, 0.37, 0.5, -0.07)
    assert np.array_equal(bits(jacobi_rowwise(g, mixed, 7)), bits(jacobi_c(g, mixed, 7)))
