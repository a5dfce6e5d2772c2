"""The reference's own acceptance batches (pkg/tests/test_acceptance.py),
recorded from the reference by tests/golden/make_acceptance_batch.py.

* criterion 1 (oracle equivalence, :132-147): the 200 configs of the batch
  (seed 20260814, domains 8..512, T 1..8, workers 1..8) — the pinned C oracle
  on CPU, and this repo's run_dtb on the B200 with the reference plan and
  with the native B200 plan, each bitwise equal to the reference's output;
* criterion 3 (capacity feasibility, :168-190): 1000 random capacity plans —
  the reference-compatible planner mirror reproduces every plan;
* criterion 4 (traffic reconciliation, :193-207): run_dtb with a reference
  plan reports exactly the reference's counters;
* criterion 6 (thread determinism, :243-257): 40 configs x threads.
"""

import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR
from paper_2306_03336_b200 import (DeviceModel, KernelConfig, StencilWeights, grid_new,
                                   plan_device_tiles, run_dtb, run_dtb_b200)
from paper_2306_03336_b200.prng import random_interior


@pytest.fixture(scope="module")
def batch():
    with open(os.path.join(GOLDEN_DIR, "acceptance_batch.json")) as fh:
        return json.load(fh)


def _grid(r):
    return grid_new(r["nx"], r["ny"], random_interior(r["nx"], r["ny"], r["seed"]))


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_batch_shape_matches_the_reference_criterion(batch):
    runs = batch["batch"]
    assert len(runs) == 200
    assert {(r["nx"], r["ny"]) for r in runs} >= {(8, 8), (512, 512)}
    assert {r["t_depth"] for r in runs} == set(range(1, 9))
    assert {r["workers"] for r in runs} == set(range(1, 9))


def test_c_oracle_reproduces_the_200_config_batch(batch, c_oracle):
    from oracle import jacobi_c
    bad = [i for i, r in enumerate(batch["batch"])
           if _sha(jacobi_c(_grid(r).data, r["weights"], r["steps"])) != r["sha256_out"]]
    assert not bad, bad


def test_planner_mirror_reproduces_criterion_3_plans(batch):
    bad = []
    for nx, ny, t, workers, elem, cap, ntiles, footprint in batch["capacity_plans"]:
        plan = plan_device_tiles((nx, ny), DeviceModel("r", workers, cap), t, elem_bytes=elem)
        if (len(plan.tiles), plan.footprint_bytes) != (ntiles, footprint) or footprint > cap:
            bad.append((nx, ny, t, workers, elem, cap))
    assert not bad, bad[:5]


@pytest.mark.gpu
def test_b200_run_dtb_reproduces_the_200_config_batch(batch):
    """Criteria 1 and 4 through this repo's run_dtb on the B200: every config
    with the reference plan (counters = the reference's) and with the native
    B200 plan (its own schedule), bitwise equal to the reference's output."""
    bad, counters = [], []
    for i, r in enumerate(batch["batch"]):
        g = _grid(r)
        w = StencilWeights(*r["weights"])
        plan = plan_device_tiles((r["nx"], r["ny"]), DeviceModel("gen", r["workers"], r["cap"]),
                                 r["t_depth"])
        assert (len(plan.tiles), plan.footprint_bytes) == (r["tiles"], r["footprint"]), i
        out, rep = run_dtb(g, w, r["steps"], plan, KernelConfig(4))
        if _sha(out.data) != r["sha256_out"]:
            bad.append((i, "reference plan"))
        if [rep.global_load_cells, rep.global_store_cells, rep.halo_exchanged_cells,
                rep.redundant_compute_cells, rep.useful_compute_cells,
                rep.scratchpad_peak_bytes, rep.elem_bytes] != r["report"]:
            counters.append(i)
        out2, rep2 = run_dtb_b200(g, w, r["steps"])
        if _sha(out2.data) != r["sha256_out"]:
            bad.append((i, "b200 plan"))
        assert rep2.useful_compute_cells == r["nx"] * r["ny"] * r["steps"]
    assert not bad, bad
    assert not counters, counters


@pytest.mark.gpu
def test_b200_thread_determinism_criterion_6(batch):
    subset = [r for r in batch["batch"] if r["nx"] <= 96 and r["ny"] <= 96][:40]
    assert len(subset) >= 20
    for r in subset:
        g = _grid(r)
        w = StencilWeights(*r["weights"])
        plan = plan_device_tiles((r["nx"], r["ny"]), DeviceModel("gen", r["workers"], r["cap"]),
                                 r["t_depth"])
        for threads in sorted({1, 2, os.cpu_count() or 1}):
            out, _ = run_dtb(g, w, r["steps"], plan, KernelConfig(4), threads=threads)
            assert _sha(out.data) == r["sha256_out"], (r["nx"], r["ny"], threads)
