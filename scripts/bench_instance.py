"""bench_single's SVD rows (pipeline.hpp:303-346) on an `nlsp gen` instance
directory — the paper's Tables 1-3 setting at N = 64 (n = 4,225) — GPU vs the
reference's own CPU code, both timed the way the reference's StopWatch times
them (host wall clock around each phase, data starting on the host).

GPU arm (this repo): libnlsp_io load_instance -> generate_smoothed_vectors
(K = 32, s1 = 10, omega = 0.66, seed = smoothing_seed(instance seed)) ->
svd_basis(rank) -> TwoLevelPreconditioner(nu1 = nu2 = 5) -> pcg(delta = 1e-6,
10 n), for ranks 4/8/16/32 (ExperimentConfig defaults, experiment.hpp:42-70).
Reference arm: the same calls through oracle/_ref (the unmodified reference
headers compiled by oracle/Makefile), one core.

With --nlss, the NLSS rows too: an (untrained) MlpModel of the default widths
(train.hpp:28-32, seed 77, bit-identical initialisation in both arms), its
basis from infer_basis (train.hpp:52-62) — the MLP forward on the device here,
the reference's forward + MGS on one core there.

With --sa, the SA row too (pipeline.hpp:316-317: sa_prolongator(A, 0.25, 0.66),
its emergent coarse dimension n_c — 2 009 at N = 64 — through the wide
kernels). The reference's SA constructor (dense MGS of n x n_c) takes minutes
at N = 64, so its arm runs SA only for n <= 1089 unless --sa-ref.

With --batch B, a throughput line per arm instead: B solves of the instance's
SVD rank-8 system (the reference harness solves its test instances
concurrently, pipeline.hpp:356) — nlsp_pcg_batch (one single-cluster solver
per system, all in one launch) vs the reference's pcg on every host core
(one single-threaded solve per core, repeated to B).

Prints one JSON line per (arm, method, rank) with smooth / inference / setup /
solve / total ms (the reference's BenchRow fields) and iterations; --reps R
repeats and keeps the median per phase.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

K, S1, OMEGA, NU, DELTA = 32, 10, 0.66, 5, 1e-6


MLP_SEED = 77


def gpu_arm(path, ranks, reps, nlss=False, with_sa=False):
    from paper_2601_20174_b200 import instance_io as io
    from paper_2601_20174_b200 import mlp
    from paper_2601_20174_b200 import nlsp
    from paper_2601_20174_b200 import sa
    ctx = nlsp.default_context()
    rows = {("SVD", r): [] for r in ranks}
    if with_sa:
        rows[("SA", 0)] = []
    if nlss:
        rows.update({("NLSS", r): [] for r in ranks})
        n0 = io.load_instance(path).matrix.dim()
        model = mlp.MlpModel.init([n0 * K] + mlp.default_hidden_widths(n0) + [n0 * K], MLP_SEED)
        model.device(ctx)
    for rep in range(reps + 1):  # rep 0 warms module loading
        t0 = time.perf_counter()
        inst = io.load_instance(path)
        t_load = time.perf_counter() - t0
        seed = mix_seed(inst.seed, 3)
        t0 = time.perf_counter()
        sv = nlsp.generate_smoothed_vectors(inst.matrix, inst.boundary_mask, K, S1, OMEGA, seed)
        ctx.synchronize()
        t_smooth = time.perf_counter() - t0
        for method, r in rows:
            t0 = time.perf_counter()
            if method == "SVD":
                p, _, _ = nlsp.svd_basis(sv.s, r)
            elif method == "SA":
                p = sa.sa_prolongator(inst.matrix, 0.25, OMEGA)
            else:
                q = mlp.infer_basis(model, sv.s)
                p = np.ascontiguousarray(q.numpy()[:, :r])  # first_cols (dense.hpp:158-164)
            ctx.synchronize()
            t_inf = time.perf_counter() - t0
            t0 = time.perf_counter()
            m = nlsp.TwoLevelPreconditioner(inst.matrix, p, OMEGA, NU, NU)
            ctx.synchronize()
            t_setup = time.perf_counter() - t0
            t0 = time.perf_counter()
            res = nlsp.pcg(inst.matrix, inst.rhs, m, DELTA, 10 * inst.matrix.dim())
            t_solve = time.perf_counter() - t0
            if rep:
                rows[(method, r)].append(dict(load=t_load, smooth=0.0 if method == "SA" else t_smooth,
                                              inference=t_inf, setup=t_setup, solve=t_solve,
                                              iterations=res.report.iterations,
                                              converged=res.report.converged, coarse_dim=m.coarse_dim()))
    return inst.matrix.dim(), rows


def ref_arm(path, ranks, reps, nlss=False, with_sa=False):
    import tempfile
    from oracle.oracle import Reference
    ref = Reference()
    rows = {("SVD", r): [] for r in ranks}
    if with_sa:
        rows[("SA", 0)] = []
    ckpt = None
    if nlss:
        rows.update({("NLSS", r): [] for r in ranks})
        n0 = ref.load_instance(path)["matrix"][0]
        from paper_2601_20174_b200 import mlp
        ckpt = os.path.join(tempfile.mkdtemp(), "model.ckpt")
        ref.mlp_create_save([n0 * K] + mlp.default_hidden_widths(n0) + [n0 * K], MLP_SEED, ckpt)
    for _ in range(reps):
        t0 = time.perf_counter()
        inst = ref.load_instance(path)
        t_load = time.perf_counter() - t0
        a = inst["matrix"]
        seed = int(ref.lib.ref_mix_seed(inst["seed"], 3))
        t0 = time.perf_counter()
        s = ref.generate_smoothed_vectors(a, inst["mask"], K, S1, OMEGA, seed)
        t_smooth = time.perf_counter() - t0
        for method, r in list(rows):
            t0 = time.perf_counter()
            if method == "SVD":
                u, _, _, _ = ref.svd(s)
                t_inf = time.perf_counter() - t0
            elif method == "SA":
                u = ref.sa_prolongator(a, 0.25, OMEGA)
                r = u.shape[1]
                t_inf = time.perf_counter() - t0
            else:
                u, ms = ref.infer_basis(ckpt, s, K)  # timed inside (checkpoint load excluded)
                t_inf = ms / 1e3
            p = np.ascontiguousarray(u[:, :r])
            t0 = time.perf_counter()
            t = ref.twolevel(a, p, OMEGA, NU, NU)
            t_setup = time.perf_counter() - t0
            t0 = time.perf_counter()
            res = ref.pcg(a, inst["rhs"], 2, t, DELTA, 10 * a[0])
            t_solve = time.perf_counter() - t0
            key = (method, 0) if method == "SA" else (method, r)
            rows[key].append(dict(load=t_load, smooth=0.0 if method == "SA" else t_smooth, inference=t_inf,
                                  setup=t_setup, solve=t_solve, iterations=res.iterations,
                                  converged=res.converged, coarse_dim=r))
    if ckpt:
        os.remove(ckpt)
    return a[0], rows


def batch_arm(arm, path, count, reps):
    import os as _os
    if arm == "gpu":
        from paper_2601_20174_b200 import instance_io as io
        from paper_2601_20174_b200 import nlsp
        ctx = nlsp.default_context()
        inst = io.load_instance(path)
        sv = nlsp.generate_smoothed_vectors(inst.matrix, inst.boundary_mask, K, S1, OMEGA, mix_seed(inst.seed, 3))
        p, _, _ = nlsp.svd_basis(sv.s, 8)
        m = nlsp.TwoLevelPreconditioner(inst.matrix, p, OMEGA, NU, NU)
        systems = [(inst.matrix, inst.rhs, m)] * count
        nlsp.pcg_batch(systems, DELTA, 10 * inst.matrix.dim())  # warm
        ts = []
        for _ in range(reps):
            ctx.synchronize()
            t0 = time.perf_counter()
            res = nlsp.pcg_batch(systems, DELTA, 10 * inst.matrix.dim())
            ts.append(time.perf_counter() - t0)
        n, iters, dev_ms = inst.matrix.dim(), res[0].report.iterations, res[0].report.solve_ms
        cores = None
    else:
        from oracle.oracle import Reference
        ref = Reference()
        inst = ref.load_instance(path)
        a = inst["matrix"]
        s = ref.generate_smoothed_vectors(a, inst["mask"], K, S1, OMEGA, int(ref.lib.ref_mix_seed(inst["seed"], 3)))
        u, _, _, _ = ref.svd(s)
        t = ref.twolevel(a, np.ascontiguousarray(u[:, :8]), OMEGA, NU, NU)
        cores = _os.cpu_count() or 1
        ts = []
        for _ in range(reps):
            done, t0 = 0, time.perf_counter()
            while done < count:
                th = min(cores, count - done)
                _, iters = ref.pcg_parallel(a, inst["rhs"], 2, t, DELTA, 10 * a[0], th)
                done += th
            ts.append(time.perf_counter() - t0)
        n, dev_ms = a[0], None
    wall = statistics.median(ts)
    return {"impl": arm, "instance": os.path.basename(path), "n": n, "method": "SVD", "rank": 8, "batch": count,
            "iterations": iters, "wall_ms": round(wall * 1e3, 3), "solves_per_s": round(count / wall, 2),
            "device_ms": dev_ms, "cores": cores, "reps": reps}


def mix_seed(seed, tag):
    # rng.hpp mix_seed through the product's host generator library
    from paper_2601_20174_b200 import _lib as L
    return int(L.inputs_lib().nlsp_mix_seed(seed, tag))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--instance", default=os.path.join(ROOT, "tests", "golden", "io", "inst_diffusion_n64"))
    ap.add_argument("--ranks", default="4,8,16,32")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--impl", choices=["gpu", "reference", "both"], default="both")
    ap.add_argument("--nlss", action="store_true", help="also the NLSS (MLP inference) rows")
    ap.add_argument("--sa", action="store_true", help="also the SA row")
    ap.add_argument("--sa-ref", action="store_true", help="run the reference SA row at any size")
    ap.add_argument("--batch", type=int, default=0, help="throughput of B concurrent solves")
    args = ap.parse_args()
    ranks = [int(r) for r in args.ranks.split(",")]
    arms = ["gpu", "reference"] if args.impl == "both" else [args.impl]
    if args.batch:
        for arm in arms:
            print(json.dumps(batch_arm(arm, args.instance, args.batch, args.reps)), flush=True)
        return
    for arm in arms:
        sa_here = args.sa
        if arm == "reference" and args.sa and not args.sa_ref:
            from paper_2601_20174_b200 import instance_io as io
            sa_here = io.load_instance(args.instance).matrix.dim() <= 1089
        n, rows = (gpu_arm if arm == "gpu" else ref_arm)(args.instance, ranks, args.reps, args.nlss, sa_here)
        for (method, r), rr in rows.items():
            med = {k: statistics.median(x[k] for x in rr) * 1e3
                   for k in ("load", "smooth", "inference", "setup", "solve")}
            out = {"impl": arm, "instance": os.path.basename(args.instance), "n": n, "method": method,
                   "rank": r if method != "SA" else rr[-1]["coarse_dim"], "K": K, "s1": S1, "nu": NU, "delta": DELTA,
                   "iterations": rr[-1]["iterations"], "converged": rr[-1]["converged"],
                   "ms": {k: round(v, 3) for k, v in med.items()},
                   "total_ms": round(med["smooth"] + med["inference"] + med["setup"] + med["solve"], 3),
                   "reps": len(rr), "cores": 1 if arm == "reference" else None}
            print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
