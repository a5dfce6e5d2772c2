"""Generate the trace fixtures from the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_trace_golden.py

It imports the reference package `dtb` (pkg/src/dtb) read-only and records
run_dtb_trace (engine.py:329-345) and jacobi_reference_trace (oracle.py:37-59)
outputs — every block's load image, superstep images and stored slice — for a
few small plans, into trace_golden.npz. Nothing at test time reads
/root/reference.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

# (name, nx, ny, workers, scratch bytes per worker, t_depth, steps, probe, valid, poison, seed,
#  ghost, weights)
CASES = [
    ("tiny2", 16, 16, 2, 2048, 2, 6, 1, None, False, 5, 0.25, (0.11, -0.2, 0.37, 0.5, -0.07)),
    ("tiny2_valid", 16, 16, 2, 2048, 2, 4, 0, (2, 3, 11, 10), False, 7, 0.5,
     (0.2, 0.2, 0.2, 0.2, 0.2)),
    ("tiny2_poison", 16, 16, 2, 2048, 2, 4, 1, None, True, 9, 0.0, (0.11, -0.2, 0.37, 0.5, -0.07)),
    ("w3_t3", 20, 14, 3, 2048, 3, 6, 2, None, False, 11, -0.5, (0.3, 0.1, 0.2, 0.1, 0.3)),
    ("w3_t3_valid_poison", 20, 14, 3, 2048, 3, 3, 1, (1, 1, 17, 12), True, 13, 0.75,
     (0.2, 0.2, 0.2, 0.2, 0.2)),
]
# (name, nx, ny, steps, stride, seed)
ORACLE_CASES = [("o_s1", 9, 7, 3, 1, 21), ("o_s2", 9, 7, 5, 2, 22), ("o_s3", 12, 5, 7, 3, 23),
                ("o_zero", 6, 6, 0, 1, 24)]


def main():
    sys.path.insert(0, REF)
    from dtb import (DeviceModel, Rect, StencilWeights, grid_new, jacobi_reference_trace,
                     plan_device_tiles, random_interior)
    from dtb.engine import run_dtb_trace

    arrays, meta = {}, {"run_dtb_trace": [], "jacobi_reference_trace": []}
    for (name, nx, ny, workers, cap, td, steps, probe, valid, poison, seed, ghost, w) in CASES:
        g = grid_new(nx, ny, random_interior(nx, ny, seed), ghost=ghost)
        plan = plan_device_tiles((nx, ny), DeviceModel("tiny", workers, cap), td)
        vr = Rect(*valid) if valid is not None else None
        out, rep, tr = run_dtb_trace(g, StencilWeights(*w), steps, plan, probe=probe, valid=vr,
                                     poison=poison)
        arrays[f"{name}_in"] = g.data
        arrays[f"{name}_out"] = out.data
        for b, blk in enumerate(tr.blocks):
            arrays[f"{name}_b{b}_load"] = blk.load
            arrays[f"{name}_b{b}_store"] = blk.store
            for s, img in enumerate(blk.steps):
                arrays[f"{name}_b{b}_s{s + 1}"] = img
        lr = tr.load_region
        meta["run_dtb_trace"].append({
            "name": name, "nx": nx, "ny": ny, "workers": workers, "cap": cap, "t_depth": td,
            "steps": steps, "probe": probe, "valid": valid, "poison": poison, "weights": list(w),
            "blocks": len(tr.blocks), "load_region": [lr.x0, lr.y0, lr.width, lr.height],
            "tiles": len(plan.tiles),
            "report": [rep.global_load_cells, rep.global_store_cells, rep.halo_exchanged_cells,
                       rep.redundant_compute_cells, rep.useful_compute_cells]})
    for (name, nx, ny, steps, stride, seed) in ORACLE_CASES:
        g = grid_new(nx, ny, random_interior(nx, ny, seed), ghost=0.25)
        snaps = jacobi_reference_trace(g, StencilWeights.diffusive(0.2), steps, stride=stride)
        arrays[f"{name}_in"] = g.data
        for i, sn in enumerate(snaps):
            arrays[f"{name}_t{i}"] = sn.data
        meta["jacobi_reference_trace"].append({"name": name, "nx": nx, "ny": ny, "steps": steps,
                                               "stride": stride, "snapshots": len(snaps)})
    np.savez_compressed(os.path.join(HERE, "trace_golden.npz"), **arrays)
    with open(os.path.join(HERE, "trace_golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    print(f"{len(arrays)} arrays")


if __name__ == "__main__":
    main()
