"""Generate the golden fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference package `dtb` (pkg/src/dtb) read-only and records
its outputs for the hot path (jacobi_reference, oracle.py:19-34; run_dtb,
engine.py:305-326; model_dtb_traffic, metrics.py:89-126; random_interior,
prng.py:45-67). The fixtures travel with the repo; nothing at test time
reads /root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    sys.path.insert(0, REF)
    import dtb
    from dtb import (DeviceModel, KernelConfig, Rect, StencilWeights, grid_new, jacobi_reference,
                     model_dtb_traffic, plan_device_tiles, random_interior, run_dtb)
    from dtb.prng import Xoshiro256StarStar

    small = {}   # name -> arrays (exact outputs, small grids)
    cases = []   # json records with hashes (larger grids)

    def rand_grid(nx, ny, seed, ghost=0.0):
        return grid_new(nx, ny, random_interior(nx, ny, seed), ghost=ghost)

    # --- KATs of the reference tests (test_kernel.py / test_oracle.py) ---
    spike = grid_new(3, 3, lambda x, y: 1.0 if (x, y) == (1, 1) else 0.0)
    all02 = StencilWeights(0.2, 0.2, 0.2, 0.2, 0.2)
    for steps in (1, 2):
        out = jacobi_reference(spike, all02, steps)
        small[f"kat_spike{steps}_in"] = spike.data
        small[f"kat_spike{steps}_w"] = np.array(all02.astuple())
        small[f"kat_spike{steps}_out"] = out.data
    for alpha in (0.25, 0.125):
        g = grid_new(8, 8, 0.8125, ghost=0.8125)
        w = StencilWeights.diffusive(alpha)
        small[f"kat_fixed{alpha}_in"] = g.data
        small[f"kat_fixed{alpha}_w"] = np.array(w.astuple())
        small[f"kat_fixed{alpha}_out"] = jacobi_reference(g, w, 20).data
    g = grid_new(4, 4, 0.8125, ghost=0.8125)
    w = StencilWeights(0.3, 0.1, 0.2, 0.1, 0.3)
    small["kat_drift_in"] = g.data
    small["kat_drift_w"] = np.array(w.astuple())
    small["kat_drift_out"] = jacobi_reference(g, w, 1).data

    # --- random small grids, exact outputs ---
    rng = Xoshiro256StarStar(424242)
    shapes = [(1, 1), (2, 3), (3, 3), (5, 4), (7, 9), (9, 7), (16, 16), (31, 17), (33, 29),
              (64, 48), (37, 41), (129, 5), (5, 131), (100, 3)]
    for i, (nx, ny) in enumerate(shapes):
        seed = rng.randint(0, 2 ** 40)
        ghost = rng.choice([0.0, 0.125, 0.75, -0.0, 1.5])
        weights = StencilWeights(*(rng.uniform(-1.0, 1.0) for _ in range(5)))
        steps = rng.choice([1, 2, 3, 4, 7, 8, 13])
        gr = rand_grid(nx, ny, seed, ghost)
        small[f"rand{i}_in"] = gr.data
        small[f"rand{i}_w"] = np.array(weights.astuple())
        small[f"rand{i}_steps"] = np.array(steps)
        small[f"rand{i}_out"] = jacobi_reference(gr, weights, steps).data

    # --- C1: 256x256 fp64, 100 steps, diffusive(0.2), seed 1 (BASELINE config 1) ---
    c1 = rand_grid(256, 256, 1)
    c1_out = jacobi_reference(c1, StencilWeights.diffusive(0.2), 100)
    cases.append({"name": "C1", "nx": 256, "ny": 256, "seed": 1, "ghost": 0.0,
                  "weights": list(StencilWeights.diffusive(0.2).astuple()), "steps": 100,
                  "sha256_out": sha(c1_out.data),
                  "samples": {f"{x},{y}": float(c1_out.data[y + 1, x + 1])
                              for x, y in [(0, 0), (128, 128), (255, 255), (17, 200)]}})
    mixed = StencilWeights(0.11, -0.2, 0.37, 0.5, -0.07)
    c1m = rand_grid(256, 256, 1, ghost=0.25)
    cases.append({"name": "C1_mixed", "nx": 256, "ny": 256, "seed": 1, "ghost": 0.25,
                  "weights": list(mixed.astuple()), "steps": 100,
                  "sha256_out": sha(jacobi_reference(c1m, mixed, 100).data)})

    # --- run_dtb: outputs + reference traffic reports for several plans ---
    runs = []
    for (nx, ny, workers, cap, t, steps, seed, ghost, valid) in [
        (8, 8, 1, 1 << 16, 1, 1, 1, 0.5, None),
        (64, 64, 2, 8192, 4, 8, 2, 0.125, None),
        (64, 64, 3, 4096, 4, 8, 3, 0.125, None),
        (33, 29, 3, 6144, 4, 8, 7, 1.5, None),
        (40, 36, 4, 8192, 4, 8, 11, 0.0, (8, 8, 24, 20)),
        (48, 48, 4, 4096, 2, 6, 4, 0.0, None),
        (3, 3, 8, 4096, 1, 2, 13, 2.0, None),
    ]:
        gr = rand_grid(nx, ny, seed, ghost)
        plan = plan_device_tiles((nx, ny), DeviceModel("d", workers, cap), t)
        v = Rect(*valid) if valid else None
        out, rep = run_dtb(gr, StencilWeights.diffusive(0.2), steps, plan, KernelConfig(4),
                           valid=v)
        assert rep == model_dtb_traffic(plan, steps, v)
        key = f"dtb{len(runs)}"
        small[f"{key}_in"] = gr.data
        small[f"{key}_out"] = out.data
        runs.append({"key": key, "nx": nx, "ny": ny, "workers": workers, "cap": cap,
                     "t_depth": t, "steps": steps, "valid": valid,
                     "tiles": len(plan.tiles), "footprint": plan.footprint_bytes,
                     "report": [rep.global_load_cells, rep.global_store_cells,
                                rep.halo_exchanged_cells, rep.redundant_compute_cells,
                                rep.useful_compute_cells, rep.scratchpad_peak_bytes,
                                rep.elem_bytes]})

    # --- acceptance 2: pruned 560x536 domain, valid 512^2, T=4, 8 steps, a100, seed 424242 ---
    padded = rand_grid(560, 536, 424242)
    valid = Rect(24, 12, 512, 512)
    problem = dtb.grid_extract(padded, valid)
    want = jacobi_reference(problem, StencilWeights.diffusive(0.2), 8)
    cases.append({"name": "pruned_560x536", "nx": 560, "ny": 536, "seed": 424242, "ghost": 0.0,
                  "weights": list(StencilWeights.diffusive(0.2).astuple()), "steps": 8,
                  "valid": [24, 12, 512, 512], "sha256_valid_out": sha(want.data)})

    # --- acceptance-1-style randomized batch (seed 20260814), hashes only ---
    batch = []
    rng = Xoshiro256StarStar(20260814)
    while len(batch) < 40:
        nx = max(8, min(512, int(8 * (512 / 8) ** rng.random())))
        ny = max(8, min(512, int(8 * (512 / 8) ** rng.random())))
        t = rng.randint(1, 8)
        steps = t * rng.choice([1, 2, 4])
        if nx * ny * steps > 600_000:
            continue
        w = StencilWeights(*(rng.uniform(-1.0, 1.0) for _ in range(5)))
        seed = rng.randint(0, 2 ** 62)
        gr = rand_grid(nx, ny, seed)
        batch.append({"nx": nx, "ny": ny, "steps": steps, "t_depth": t, "seed": seed,
                      "weights": list(w.astuple()),
                      "sha256_out": sha(jacobi_reference(gr, w, steps).data)})

    # --- prng frozen vectors ---
    prng = {"splitmix64_1234567": [int(v) for v in dtb.splitmix64(1234567, 5)],
            "random_interior_3x2_seed9": random_interior(3, 2, 9).tolist()}

    np.savez_compressed(os.path.join(HERE, "golden_small.npz"), **small)
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_golden.py",
                   "reference": "arxiv/paper_2306_03336 pkg/src/dtb " + dtb.__version__,
                   "cases": cases, "runs": runs, "batch": batch, "prng": prng}, fh, indent=1)
    print("wrote", len(small), "arrays,", len(cases), "cases,", len(runs), "runs,",
          len(batch), "batch")


if __name__ == "__main__":
    main()
