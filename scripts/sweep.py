#!/usr/bin/env python3
"""Config 4: shape sweep 256..8192 (square, tall-skinny, wide), several strategy
trees per shape, one B200. Device time per launch with the L2 flushed before
every launch: one CUDA-event pair around R x (flush + launch) minus one around
R x flush, over R (single-launch event pairs step in ~2 us quanta on the B200
box, profiles/round2/experiments.txt); median of `--steps` such sequences.
Writes profiles/<tag>_sweep.json and prints a table.

  python scripts/sweep.py [--tag round1] [--quick]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2003_06324_b200 as fi  # noqa: E402

SQUARE = [256, 512, 1024, 2048, 4096, 8192]
TALL = [(4096, 256, 4096), (4096, 512, 4096), (8192, 256, 8192), (8192, 512, 8192)]
WIDE = [(256, 4096, 4096), (512, 4096, 4096), (256, 8192, 8192), (512, 8192, 8192)]


def peak():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    except Exception:
        return 1590.0


def per_launch_ms(fn, steps, flush, R=20):
    """Median over `steps` of (R x (flush + fn) - R x flush) / R, in ms."""
    s = torch.cuda.current_stream()

    def seq(f):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        for _ in range(R):
            flush.zero_()
            if f:
                f()
        e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1)

    seq(fn)
    ts = []
    for _ in range(steps):
        base = seq(None)
        ts.append((seq(fn) - base) / R)
    return statistics.median(ts)


def time_plan(plan, steps, flush):
    m, n, k = plan.m, plan.n, plan.k
    (ar, ac, arow), (br, bc, brow), (cr, cc, crow) = plan.shapes()
    el = {0: torch.float32, 1: torch.float16, 2: torch.bfloat16}
    A = torch.rand(ar * ac, device="cuda").to(el[plan.info.elem_a]) - 0.5
    B = torch.rand(br * bc, device="cuda").to(el[plan.info.elem_b]) - 0.5
    C = torch.empty(cr * cc, device="cuda", dtype=el[plan.info.elem_c])
    s = torch.cuda.current_stream()
    for _ in range(3):
        plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream)
    return per_launch_ms(lambda: plan.launch(A.data_ptr(), B.data_ptr(), C.data_ptr(), s.cuda_stream), steps, flush)


def time_cublas(m, n, k, steps, flush, out_dtype=torch.float32):
    """Library reference (not part of the product): cuBLAS through torch.mm on
    the same col-major problem, f16 in / f32 accumulate / f32 (or f16) out."""
    a = torch.rand((k, m), device="cuda").half() - 0.5   # col-major A = row-major A^T
    b = torch.rand((n, k), device="cuda").half() - 0.5
    if out_dtype == torch.float16:
        f = lambda: torch.mm(b, a)                          # C^T (N x M) row-major = C col-major
    else:
        f = lambda: torch.mm(b, a, out_dtype=out_dtype)
    for _ in range(3):
        f()
    return per_launch_ms(f, steps, flush)


def candidates(m, n, k, quick):
    c = dict(fi.strategies.sweep_strategies(m, n, k))
    if not quick and m * n * k <= 1024 ** 3 and m % 128 == 0 and n % 128 == 0 and k % 8 == 0:
        c["fma_listing2"] = fi.strategies.listing2(m, n, k)   # CUDA-core correctness fallback
    if not quick and m % 128 == 0 and n % 128 == 0 and k % 128 == 0 and m * n * k <= 2048 ** 3:
        c["wmma_paper"] = fi.strategies.wmma_decomp(m, n, k)  # the paper's WMMA strategy
    return c


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", default="round1")
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    flush = torch.empty(128 << 20, device="cuda")
    pk = peak()
    shapes = [(s, s, s, "square") for s in SQUARE] + [(*t, "tall") for t in TALL] + [(*w, "wide") for w in WIDE]
    results = []
    for m, n, k, kind in shapes:
        row = {"m": m, "n": n, "k": k, "kind": kind, "flops": 2.0 * m * n * k, "strategies": {}}
        for name, script in candidates(m, n, k, args.quick).items():
            try:
                plan = fi.Plan(script)
                ms = time_plan(plan, args.steps, flush)
                tf = row["flops"] / ms / 1e9
                row["strategies"][name] = {"ms": ms, "tflops": tf, "pct_peak": 100 * tf / pk, "kind": plan.kind,
                                           "streamk": int(plan.info.streamk), "ctas": int(plan.info.launch_ctas)}
            except Exception as e:  # noqa: BLE001
                row["strategies"][name] = {"error": str(e)[:200]}
        for key, odt in (("cublas_f32out", torch.float32), ("cublas_f16out", torch.float16)):
            try:
                ms = time_cublas(m, n, k, args.steps, flush, odt)
                row[key] = {"ms": ms, "tflops": row["flops"] / ms / 1e9}
            except Exception as e:  # noqa: BLE001
                row[key] = {"error": str(e)[:200]}
        ok = {k2: v for k2, v in row["strategies"].items() if "tflops" in v}
        if ok:
            best = max(ok, key=lambda x: ok[x]["tflops"])
            row["best"] = best
            row["best_tflops"] = ok[best]["tflops"]
            ai = row["flops"] / (2 * (m * k + k * n) + 4 * m * n)
            row["ceiling_tflops"] = min(pk, ai * 6531.6e9 / 1e12)
        results.append(row)
        print(f"{kind:6s} {m:5d}x{n:5d}x{k:5d}  best {row.get('best', '-'):24s} {row.get('best_tflops', 0):8.1f} TF"
              f"  (ceiling {row.get('ceiling_tflops', 0):7.1f}, cuBLAS f32/f16 out {row['cublas_f32out'].get('tflops', 0):7.1f}"
              f"/{row['cublas_f16out'].get('tflops', 0):7.1f})  " +
              "  ".join(f"{a}={v.get('tflops', float('nan')):.0f}" for a, v in row["strategies"].items()),
              flush=True)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    with open(os.path.join(ROOT, "profiles", f"{args.tag}_sweep.json"), "w") as f:
        json.dump({"peak_tflops": pk, "l2": "flushed before every timed launch",
                   "timing": "per launch: (20 x (flush + launch) - 20 x flush) / 20, median of 5 sequences",
                   "results": results}, f, indent=1)


if __name__ == "__main__":
    main()
