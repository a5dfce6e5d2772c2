"""Rewrite the bench tables of profiles/README.md, DESIGN.md and README.md from
the committed bench lines (profiles/r01/bench_*.json) and ncu summary."""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
B = {}
for w in ["c1", "c2", "c3a", "c3b", "c4", "c5", "ref"]:
    with open(os.path.join(ROOT, "profiles", "r01", f"bench_{w}.json")) as fh:
        B[w] = json.loads(fh.read().strip().splitlines()[-1])
N = json.load(open(os.path.join(ROOT, "profiles", "r01", "ncu_summary.json")))


def v(w):
    return B[w]["value"]


def e(w):
    return (B[w].get("e2e") or {}).get("value") or 0


def fr(w, k):
    return B[w]["rooflines"][k]["frac"]


def rewrite(path, rules):
    with open(path) as fh:
        lines = fh.read().split("\n")
    for i, line in enumerate(lines):
        for prefix, new in rules:
            if line.startswith(prefix):
                lines[i] = new
    s = "\n".join(lines)
    with open(path, "w") as fh:
        fh.write(s)
    return s


res = N["resident_kernel<double,4,8,0>"]
pip = N["pipe_kernel<double,4,16,4,0>"]
rewrite(os.path.join(ROOT, "profiles", "README.md"), [
    ("| **C2** fp64", f"| **C2** fp64 1900², 10⁴ steps (headline) | resident, h=4, 16×9 tiles of 128×226, 8 warps | **{v('c2'):.1f}** | {e('c2'):.1f} | smem {fr('c2','smem'):.3f} (16 B/cell vs 34.8 TB/s LDS.128), FP64 pipe {fr('c2','fp_pipe'):.3f} |"),
    ("| C1 fp64", f"| C1 fp64 256², 100 steps | resident (138 tiles, h=10) | {v('c1'):.1f} | {e('c1'):.1f} | latency-floored: ~1.25 µs per step for any tiling (`DTB_MAX_TILES` sweep); per the phase trace each two-step sweep costs ~2,000 cycles of ramp (pre-read, barrier, register-pipeline fill and drain) on top of ~200 cycles per band row, and C1's bands are 4 rows |"),
    ("| C3a fp32", f"| C3a fp32 2700², 10⁴ steps | resident, 11×13 tiles of 256×226 | {v('c3a'):.1f} | {e('c3a'):.1f} | smem {fr('c3a','smem'):.3f}, FP32 pipe {fr('c3a','fp_pipe'):.3f} |"),
    ("| C3b fp32", f"| C3b fp32 8192², 10³ steps | pipe, h=8, 35×16 segments | {v('c3b'):.1f} | {e('c3b'):.1f} | FP32 pipe {fr('c3b','fp_pipe'):.3f}, HBM {fr('c3b','hbm'):.3f} |"),
    ("| C4 fp64", f"| C4 fp64 16384², 10³ steps | pipe, h=8, 147×4 segments | {v('c4'):.1f} | {e('c4'):.1f} | FP64 pipe {fr('c4','fp_pipe'):.3f}, HBM {fr('c4','hbm'):.3f} |"),
    ("| C5 fp64", f"| C5 fp64 32768×4096 per GPU (N=1 of the weak series) | slab + pipe | {v('c5'):.1f} | — | FP64 pipe {fr('c5','fp_pipe'):.3f} |"),
    ("| reference CPU port", f"| reference CPU port (C restatement of `jacobi_reference`, pthreads, 16 host threads; `bench.py --impl reference`) | — | {v('ref'):.1f} | — | — |"),
    ("C2 GPU/CPU ratio", f"C2 GPU/CPU ratio ≈ {v('c2') / v('ref'):.0f}× against the reference's algorithm on all 16 host"),
    ("| resident_kernel<double,4,8> |", f"| resident_kernel<double,4,8> | C2 geometry, 2000 steps | {res['fp64_pipe_active_pct']:.1f} % | {res['issue_active_pct']:.1f} % | 8 | {int(res['registers_per_thread'])} | {(res['dram_bytes_read'] + res['dram_bytes_write']) / 1e6:.1f} MB (input + output; the exchange stays in L2) |"),
    ("| pipe_kernel<double,4,16,4> |", f"| pipe_kernel<double,4,16,4> | C4, one 8-step pass | {pip['fp64_pipe_active_pct']:.1f} % | {pip['issue_active_pct']:.1f} % | 16 | {int(pip['registers_per_thread'])} | {(pip['dram_bytes_read'] + pip['dram_bytes_write']) / 1e9:.2f} GB (= 1.0 read + 1.0 write of the 2.15 GB grid) |"),
])
rewrite(os.path.join(ROOT, "DESIGN.md"), [
    ("| C2 fp64 1900² ×10⁴ (headline)", f"| C2 fp64 1900² ×10⁴ (headline) | {v('c2'):.1f} (e2e {e('c2'):.1f}) | {fr('c2','fp_pipe'):.2f} (smem roofline {fr('c2','smem'):.2f}) | resident; h=4 forced by capacity, exchange every 4 steps |"),
    ("| C1 fp64 256² ×100", f"| C1 fp64 256² ×100 | {v('c1'):.1f} (e2e {e('c1'):.1f}) | {fr('c1','fp_pipe'):.2f} | resident; latency floor: each two-step band sweep has a ~2,000-cycle ramp (pre-read, barrier, pipeline fill/drain) however few rows a band has, ~1.25 µs per step for any tiling |"),
    ("| C3a fp32 2700² ×10⁴", f"| C3a fp32 2700² ×10⁴ | {v('c3a'):.1f} | {fr('c3a','fp_pipe'):.2f} | resident |"),
    ("| C3b fp32 8192² ×10³", f"| C3b fp32 8192² ×10³ | {v('c3b'):.1f} | {fr('c3b','fp_pipe'):.2f} | pipe |"),
    ("| C4 fp64 16384² ×10³", f"| C4 fp64 16384² ×10³ | {v('c4'):.1f} | {fr('c4','fp_pipe'):.2f} | pipe |"),
    ("| C5 fp64 32768×4096/GPU", f"| C5 fp64 32768×4096/GPU | {v('c5'):.1f} (N=1) | {fr('c5','fp_pipe'):.2f} | slab + pipe |"),
    ("| CPU reference port", f"| CPU reference port (C, 16 host threads) | {v('ref'):.1f} | — | ~{v('c2') / v('ref'):.0f}× below C2 (the single-threaded numpy reference: 0.11) |"),
])
p = os.path.join(ROOT, "README.md")
s = open(p).read()
s = re.sub(r"\| C2 fp64 1900², 10⁴ steps, resident \(headline\) \| [^|]*\|", f"| C2 fp64 1900², 10⁴ steps, resident (headline) | {v('c2'):.0f} (e2e {e('c2'):.0f}) |", s)
s = re.sub(r"\| C3a fp32 2700², resident \| [^|]*\|", f"| C3a fp32 2700², resident | {v('c3a'):.0f} |", s)
s = re.sub(r"\| C3b fp32 8192², pipelined streaming \| [^|]*\|", f"| C3b fp32 8192², pipelined streaming | {v('c3b'):.0f} |", s)
s = re.sub(r"\| C4 fp64 16384², pipelined streaming \| [^|]*\|", f"| C4 fp64 16384², pipelined streaming | {v('c4'):.0f} |", s)
s = re.sub(r"\| CPU: the reference.s algorithm on 16 host cores \| [^|]*\|", f"| CPU: the reference's algorithm on 16 host cores | {v('ref'):.0f} |", s)
open(p, "w").write(s)
print("tables updated: C2", round(v("c2"), 1))
