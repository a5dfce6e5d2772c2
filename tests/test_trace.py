"""run_dtb_trace / jacobi_reference_trace (engine.py:329-345, oracle.py:37-59)
against fixtures recorded from the reference itself (tests/golden/
make_trace_golden.py). Tolerance: none — images are compared as uint64 bit
patterns (NaN poison included).

CPU tests pin the host-side image assembly (the reference schedule's
double-buffer semantics) on oracle-computed states; GPU tests run the B200
entry points end to end.
"""

import json
import os

import numpy as np
import pytest

from oracle import jacobi_numpy
from paper_2306_03336_b200 import (DeviceModel, Grid2D, Rect, StencilWeights, j2d5pt_trace,
                                   plan_device_tiles, run_dtb, run_dtb_trace)
from paper_2306_03336_b200.engine import _superstep_image

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def fx():
    with open(os.path.join(HERE, "trace_golden.json")) as fh:
        meta = json.load(fh)
    return meta, dict(np.load(os.path.join(HERE, "trace_golden.npz")))


def bits(a):
    return np.ascontiguousarray(a).view(np.uint64)


def same(a, b):
    return a.shape == b.shape and np.array_equal(bits(a), bits(b))


def _plan(c):
    return plan_device_tiles((c["nx"], c["ny"]), DeviceModel("tiny", c["workers"], c["cap"]),
                             c["t_depth"])


def _states_oracle(data, c, w, steps):
    """Padded grids after 0..steps oracle steps; with a valid rect the cells
    outside it stay frozen (a jacobi of the valid block and its 1-cell ring)."""
    out = [data.copy()]
    v = c["valid"]
    for _ in range(steps):
        cur = out[-1].copy()
        if v is None:
            cur = jacobi_numpy(cur, w, 1)
        else:
            x0, y0, wd, ht = v
            sub = cur[y0:y0 + ht + 2, x0:x0 + wd + 2]
            cur[y0:y0 + ht + 2, x0:x0 + wd + 2] = jacobi_numpy(sub, w, 1)
        out.append(cur)
    return out


def test_image_assembly_matches_reference_on_oracle_states(fx):
    meta, arr = fx
    for c in meta["run_dtb_trace"]:
        name, td = c["name"], c["t_depth"]
        plan = _plan(c)
        assert len(plan.tiles) == c["tiles"]
        tile = plan.tiles[c["probe"]]
        load = tile.load_region
        assert [load.x0, load.y0, load.width, load.height] == c["load_region"]
        valid = Rect(*c["valid"]) if c["valid"] else Rect(0, 0, c["nx"], c["ny"])
        states = _states_oracle(arr[f"{name}_in"], c, tuple(c["weights"]), c["steps"])
        for b in range(c["blocks"]):
            blk = states[b * td:(b + 1) * td + 1]
            base = blk[0][load.y0 + 1:load.y1 + 1, load.x0 + 1:load.x1 + 1]
            assert same(base, arr[f"{name}_b{b}_load"]), (name, b)
            for s in range(1, td + 1):
                img = _superstep_image(base, load, blk, s, tile, valid, c["poison"])
                assert same(img, arr[f"{name}_b{b}_s{s}"]), (name, b, s)
        assert same(states[-1], arr[f"{name}_out"]), name


@pytest.mark.gpu
def test_run_dtb_trace_matches_reference(fx):
    meta, arr = fx
    for c in meta["run_dtb_trace"]:
        name = c["name"]
        g = Grid2D(c["nx"], c["ny"], arr[f"{name}_in"])
        w = StencilWeights(*c["weights"])
        plan = _plan(c)
        valid = Rect(*c["valid"]) if c["valid"] else None
        out, rep, tr = run_dtb_trace(g, w, c["steps"], plan, probe=c["probe"], valid=valid,
                                     poison=c["poison"])
        assert tr.tile_index == c["probe"]
        assert [tr.load_region.x0, tr.load_region.y0, tr.load_region.width,
                tr.load_region.height] == c["load_region"]
        assert len(tr.blocks) == c["blocks"]
        for b, blk in enumerate(tr.blocks):
            assert same(blk.load, arr[f"{name}_b{b}_load"]), (name, b)
            assert same(blk.store, arr[f"{name}_b{b}_store"]), (name, b)
            assert len(blk.steps) == c["t_depth"]
            for s, img in enumerate(blk.steps):
                assert same(img, arr[f"{name}_b{b}_s{s + 1}"]), (name, b, s + 1)
        assert same(out.data, arr[f"{name}_out"]), name
        assert [rep.global_load_cells, rep.global_store_cells, rep.halo_exchanged_cells,
                rep.redundant_compute_cells, rep.useful_compute_cells] == c["report"]
        # the traced solve and the plain one agree
        plain, _ = run_dtb(g, w, c["steps"], plan, valid=valid, poison=c["poison"])
        assert same(plain.data, out.data)


@pytest.mark.gpu
def test_run_dtb_trace_probe_bounds(fx):
    meta, arr = fx
    c = meta["run_dtb_trace"][0]
    g = Grid2D(c["nx"], c["ny"], arr[f"{c['name']}_in"])
    plan = _plan(c)
    for probe in (len(plan.tiles), -1):
        with pytest.raises(IndexError):
            run_dtb_trace(g, StencilWeights.diffusive(0.2), 2, plan, probe=probe)
    with pytest.raises(ValueError):  # not a multiple of t_depth
        run_dtb_trace(g, StencilWeights.diffusive(0.2), 3, plan, probe=0)


@pytest.mark.gpu
def test_j2d5pt_trace_matches_jacobi_reference_trace(fx):
    meta, arr = fx
    for c in meta["jacobi_reference_trace"]:
        name = c["name"]
        g = Grid2D(c["nx"], c["ny"], arr[f"{name}_in"])
        snaps = j2d5pt_trace(g, StencilWeights.diffusive(0.2), c["steps"], stride=c["stride"])
        assert len(snaps) == c["snapshots"], name
        for i, sn in enumerate(snaps):
            assert same(sn.data, arr[f"{name}_t{i}"]), (name, i)


def test_j2d5pt_trace_argument_errors():
    g = Grid2D(4, 4, np.zeros((6, 6)))
    with pytest.raises(ValueError):
        j2d5pt_trace(g, StencilWeights.diffusive(0.2), 2, stride=0)
    with pytest.raises(ValueError):
        j2d5pt_trace(g, StencilWeights.diffusive(0.2), -1)
