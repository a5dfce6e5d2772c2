"""Record the reference's own acceptance batches as golden data.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_acceptance_batch.py

Restates the sampler of the reference's acceptance suite exactly
(/root/reference/pkg/tests/test_acceptance.py:59-73 `_sample_dim` /
`_sample_capacity`, :95-129 the `batch` fixture: seed 20260814, two pinned
corners, then rejection-sampled configs until 200) and of its criterion 3
(:168-190: seed 20260815, 1000 random capacity plans), drawing from the
reference's own Xoshiro256StarStar, scratchpad_footprint and
plan_device_tiles, and records what the REFERENCE computes for each config:
the sha256 of jacobi_reference's output (equal to run_dtb's, which the
reference asserts), the reference run_dtb TrafficReport, and the plan
(tile count, footprint). The GPU test replays the batch through this repo's
run_dtb on the B200; the CPU test replays criterion 3 through the
reference-compatible planner mirror. Nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

BATCH_SEED = 20260814
N_CONFIGS = 200


def main():
    sys.path.insert(0, REF)
    import dtb
    from dtb import (DeviceModel, KernelConfig, StencilWeights, grid_new, jacobi_reference,
                     model_dtb_traffic, plan_device_tiles, random_interior, run_dtb)
    from dtb.planner import scratchpad_footprint
    from dtb.prng import Xoshiro256StarStar

    def sample_dim(rng):  # test_acceptance.py:59-60
        return max(8, min(512, int(8 * (512 / 8) ** rng.random())))

    def sample_capacity(rng, nx, ny, t_depth, workers):  # test_acceptance.py:63-73
        lo = scratchpad_footprint(
            (min(1 + 2 * t_depth, nx + 2), min(1 + 2 * t_depth, ny + 2)), t_depth, 8, workers)
        hi = scratchpad_footprint(
            (min(nx + 2 * t_depth, nx + 2), min(ny + 2 * t_depth, ny + 2)), t_depth, 8, workers)
        if hi <= lo:
            return lo
        return max(lo, int(lo * (hi / lo) ** rng.random()))

    t0 = time.perf_counter()
    records = []

    def execute(nx, ny, t_depth, steps, workers, cap, weights, seed):  # :76-92
        plan = plan_device_tiles((nx, ny), DeviceModel("gen", workers, cap), t_depth)
        grid = grid_new(nx, ny, random_interior(nx, ny, seed))
        result, report = run_dtb(grid, weights, steps, plan, KernelConfig(4))
        want = jacobi_reference(grid, weights, steps)
        assert result.data.tobytes() == want.data.tobytes()
        assert report == model_dtb_traffic(plan, steps)
        records.append({
            "nx": nx, "ny": ny, "t_depth": t_depth, "steps": steps, "workers": workers,
            "cap": cap, "weights": list(weights.astuple()), "seed": seed,
            "tiles": len(plan.tiles), "footprint": plan.footprint_bytes,
            "report": [report.global_load_cells, report.global_store_cells,
                       report.halo_exchanged_cells, report.redundant_compute_cells,
                       report.useful_compute_cells, report.scratchpad_peak_bytes,
                       report.elem_bytes],
            "sha256_out": hashlib.sha256(want.data.tobytes()).hexdigest(),
        })

    rng = Xoshiro256StarStar(BATCH_SEED)
    for nx, ny, t_depth, steps, workers in [(512, 512, 8, 8, 8), (8, 8, 1, 4, 1)]:  # :101-110
        cap = sample_capacity(rng, nx, ny, t_depth, workers)
        weights = StencilWeights(*(rng.uniform(-1.0, 1.0) for _ in range(5)))
        execute(nx, ny, t_depth, steps, workers, cap, weights, rng.randint(0, 2 ** 62))
    while len(records) < N_CONFIGS:  # :112-127
        nx, ny = sample_dim(rng), sample_dim(rng)
        t_depth = rng.randint(1, 8)
        steps = t_depth * rng.choice([1, 2, 4])
        workers = rng.randint(1, 8)
        if nx * ny * steps > 1_200_000:
            continue
        cap = sample_capacity(rng, nx, ny, t_depth, workers)
        plan = plan_device_tiles((nx, ny), DeviceModel("gen", workers, cap), t_depth)
        blocks = steps // t_depth
        if len(plan.tiles) * blocks * (2 * t_depth + 2) * workers > 40_000:
            continue
        weights = StencilWeights(*(rng.uniform(-1.0, 1.0) for _ in range(5)))
        execute(nx, ny, t_depth, steps, workers, cap, weights, rng.randint(0, 2 ** 62))

    # criterion 3 (:168-190): 1000 random plans must respect the capacity
    plans = []
    rng = Xoshiro256StarStar(BATCH_SEED + 1)
    for _ in range(1000):
        nx = rng.randint(1, 128)
        ny = rng.randint(1, 128)
        t_depth = rng.randint(1, 16)
        workers = rng.randint(1, 128)
        elem = rng.choice([4, 8])
        lo = scratchpad_footprint((min(1 + 2 * t_depth, nx + 2), min(1 + 2 * t_depth, ny + 2)),
                                  t_depth, elem, workers)
        cap = lo + rng.randint(0, 4 * lo)
        plan = plan_device_tiles((nx, ny), DeviceModel("r", workers, cap), t_depth,
                                 elem_bytes=elem)
        assert plan.footprint_bytes <= cap
        plans.append([nx, ny, t_depth, workers, elem, cap, len(plan.tiles),
                      plan.footprint_bytes])

    with open(os.path.join(HERE, "acceptance_batch.json"), "w") as fh:
        json.dump({"generator": "tests/golden/make_acceptance_batch.py",
                   "reference": "arxiv/paper_2306_03336 pkg/src/dtb " + dtb.__version__,
                   "sampler": "pkg/tests/test_acceptance.py:59-129 (seed 20260814), "
                              ":168-190 (seed 20260815)",
                   "batch": records, "capacity_plans": plans}, fh)
    print(f"{len(records)} batch configs, {len(plans)} capacity plans, "
          f"{time.perf_counter() - t0:.1f}s")


if __name__ == "__main__":
    main()
