"""Full forward + inverse SHT at N=4096 (BASELINE config 3) on ONE B200.

The plan (~370 GB of payload at tol 1e-10) does not fit one GPU, so the
transform runs through ChunkedSht (paper_2004_11346_b200/ooc.py): orders
planned / packed / uploaded / applied chunk by chunk, the φ DFT once over
all rows.  Prints one JSON line and writes it to gpurun_out/ooc_n<N>.json.

Checks (CPU oracle, tests-only code, imported here as the checker):
  * sampled orders: GPU forward ALT (assembled from the θ-major node
    halves) vs oracle.apply.alt_forward on the same factors, <= 1e-12;
  * sampled row pairs: the GPU grid rows vs a numpy restatement of the
    synthesis (sht.py:137-148) on the GPU's own node halves, <= 1e-12;
  * sampled orders: GPU inverse coefficients vs the oracle's transposed
    half applies on the GPU's own analysis folds, <= 1e-12 (and, for
    information, vs oracle alt_inverse of a numpy spectrum column);
  * round trip coefficients -> grid -> coefficients (relative l2).
CPU baseline: oracle forward + inverse ALT of the sampled orders on one
core, extrapolated by payload values to all orders (stated as such).
"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--chunks", type=int, default=24)
    ap.add_argument("--procs", type=int, default=0)
    ap.add_argument("--samples", default="1,2048,5000,8191")
    ap.add_argument("--rows", default="0,1000,4095")
    ap.add_argument("--reserve-gb", type=float, default=24.0)
    ap.add_argument("--out", default="gpurun_out/ooc_n{n}.json")
    ap.add_argument("--only", default="",
                    help="process only these chunks (comma list): a sampled run "
                         "through the full grid and DFT stage (N=8192)")
    ap.add_argument("--decay", type=float, default=1.0,
                    help="coefficient spectrum (1+k)^-decay (config 5: 2)")
    ap.add_argument("--real-grid", action="store_true",
                    help="also time an inverse of a real iid U(-1,1) grid (config 5)")
    ap.add_argument("--oracle-all", action="store_true",
                    help="global parity: run the oracle's ALT on EVERY order as each chunk "
                         "is planned (forward, and inverse on a pocketfft spectrum of the "
                         "GPU grid); implies no resident chunks (all replanned)")
    ap.add_argument("--oracle-threads", type=int, default=0)
    ap.add_argument("--regen", type=float, default=0.0,
                    help="fraction of full-height turning tiles regenerated on the GPU "
                         "(f1): smaller resident chunks")
    args = ap.parse_args()

    import torch
    from threadpoolctl import threadpool_limits
    from bench import synthetic_coeffs
    from paper_2004_11346_b200 import SamplingConfig, plan_alt
    from paper_2004_11346_b200.ooc import ChunkedSht
    import oracle.apply as OA

    n = args.n
    L = 4 * n - 1
    params = SamplingConfig(tolerance=args.tol)
    t0 = time.perf_counter()
    only = [int(v) for v in args.only.split(",") if v] or None

    # --oracle-all: the CPU oracle (oracle/apply.py = the reference's
    # alt_forward / alt_inverse on the same factors) runs on every order
    # while its chunk's plans are on the host; the phi stage is numpy's
    # pocketfft, as in sht.py:148,161
    ora = {"fwd_buf": None, "spectrum": None, "back": None, "seconds": 0.0}

    def oracle_chunk(plans):
        from concurrent.futures import ThreadPoolExecutor
        _, offs_ = OA.coeff_offsets(n)
        phi0_ = np.pi / L

        def one(p):
            m = p.m
            with threadpool_limits(limits=1):
                for mm in ((m, -m) if m else (m,)):
                    i = (2 * n - 1) + mm
                    if ora["spectrum"] is None:
                        g = OA.alt_forward(p, flat[offs_[i]:offs_[i + 1]])
                        ora["fwd_buf"][:, mm % L] = g * np.exp(1j * mm * phi0_)
                    else:
                        col = ora["spectrum"][:, mm % L] * np.exp(-1j * mm * phi0_)
                        ora["back"][offs_[i]:offs_[i + 1]] = OA.alt_inverse(p, col)

        t = time.perf_counter()
        with ThreadPoolExecutor(args.oracle_threads or (os.cpu_count() or 1)) as ex:
            list(ex.map(one, plans))
        ora["seconds"] += time.perf_counter() - t

    planner = None
    if args.oracle_all:
        from paper_2004_11346_b200 import plan_orders
        from paper_2004_11346_b200.legendre import gauss_legendre
        q_all = gauss_legendre(2 * n)
        ora["fwd_buf"] = np.zeros((2 * n, L), dtype=np.complex128)

        def planner(orders):
            plans = plan_orders(n, orders, params, processes=args.procs, quadrature=q_all)
            oracle_chunk(plans)
            return plans
        args.reserve_gb = 1e6   # no resident chunks: every inverse chunk is replanned
    _, offs0 = OA.coeff_offsets(n)
    if args.oracle_all:
        if only is not None or args.decay != 1.0:
            raise SystemExit("--oracle-all is for the whole C3 transform")
        flat = synthetic_coeffs(n, seed=3)
    run = ChunkedSht(n, args.chunks, params=params, processes=args.procs,
                     reserve_bytes=int(args.reserve_gb * (1 << 30)), verbose=True, only=only,
                     planner=planner, regen=args.regen)
    if args.oracle_all:
        # the context plan (order 2N-1) went through the planner too
        ora["fwd_buf"][:] = 0.0
    if only is None and args.decay == 1.0:
        flat = synthetic_coeffs(n, seed=3)
        subset = None
    else:
        # coefficients (iid N(0,1) (1+k)^-decay) on the processed orders only
        subset = sorted(m for c in (only or range(len(run.chunks))) for m in run.chunks[c])
        flat = np.zeros(int(offs0[-1]), dtype=np.complex128)
        rng = np.random.default_rng(3)
        for m in subset:
            for mm in ((m, -m) if m else (m,)):
                i = (2 * n - 1) + mm
                k = np.arange(abs(mm), 2 * n, dtype=np.float64)
                flat[offs0[i]:offs0[i + 1]] = (rng.standard_normal(k.size)
                                               + 1j * rng.standard_normal(k.size)) / (1.0 + k) ** args.decay
    grid = torch.empty((2 * n, L), dtype=torch.complex128, device="cuda")
    fwd = run.forward(flat, grid)
    if args.oracle_all:
        t = time.perf_counter()
        want_grid = L * np.fft.ifft(ora["fwd_buf"], axis=1)
        ora["fwd_buf"] = None
        hg = grid.cpu().numpy()
        rows = np.linalg.norm(hg - want_grid, axis=1) / np.linalg.norm(want_grid, axis=1)
        ora_res = {"fwd_rel_l2": float(np.linalg.norm(hg - want_grid) / np.linalg.norm(want_grid)),
                   "fwd_worst_row": float(rows.max())}
        del want_grid
        ora["spectrum"] = np.fft.fft(hg, axis=1) / L
        ora["back"] = np.zeros(int(offs0[-1]), dtype=np.complex128)
        del hg
        ora["seconds"] += time.perf_counter() - t
    print(f"forward: device {fwd['device_ms']:.1f} ms (ALT {fwd['alt_ms']:.1f} ms, "
          f"{fwd['alt_gbs']:.0f} GB/s), plan {fwd['plan_s']:.0f} s, "
          f"pack+upload {fwd['pack_upload_s']:.0f} s", file=sys.stderr, flush=True)

    samples = [int(v) for v in args.samples.split(",") if v]
    if subset is not None:
        samples = [m for m in samples if m in set(subset)] or \
            [subset[0], subset[len(subset) // 2], subset[-1]]
    checks = {}
    _, offs = OA.coeff_offsets(n)
    plans = {}
    cpu = {"seconds": 0.0, "values": 0}
    with threadpool_limits(limits=1):
        for m in samples:
            plans[m] = p = plan_alt(n, m, params, quadrature=run.quadrature)
    # forward ALT of sampled orders from the θ-major buffer
    errs = []
    for m in samples:
        e = run.node_entries(m)
        g_o, g_e = e[0], e[1]
        full = np.concatenate([(g_e - g_o)[::-1], g_e + g_o])
        for sgn, cols in ((1, (0, 1)), (-1, (2, 3))):
            if m == 0 and sgn < 0:
                continue
            i = (2 * n - 1) + sgn * m
            beta = flat[offs[i]:offs[i + 1]]
            with threadpool_limits(limits=1):
                t = time.perf_counter()
                want = OA.alt_forward(plans[m], beta)
                cpu["seconds"] += time.perf_counter() - t
            got = full[:, cols[0]] + 1j * full[:, cols[1]]
            errs.append(float(np.linalg.norm(got - want) / np.linalg.norm(want)))
    checks["alt_forward_vs_oracle_max"] = max(errs)
    # synthesis of sampled row pairs on the GPU's node halves
    phi0 = np.pi / L
    yb = run.ybuf.cpu().numpy()
    lay = run.layout
    ms = np.arange(2 * n)
    errs = []
    for r in sorted({min(int(v), n - 1) for v in args.rows.split(",") if v}):
        spec = np.zeros((2, L), dtype=np.complex128)   # rows n+r, n-1-r
        ent = np.zeros((2, 2 * n, 4))
        for par in range(2):
            h = lay[2 * ms + par]
            ok = h["ncols"] > 0
            idx = h["y"][ok].astype(np.int64) + r * h["x"][ok].astype(np.int64)
            ent[par][ok] = yb[idx]
        go, ge = ent[0], ent[1]
        for row, v in ((0, ge + go), (1, ge - go)):
            plus = v[:, 0] + 1j * v[:, 1]
            minus = v[:, 2] + 1j * v[:, 3]
            spec[row, ms] = plus * np.exp(1j * ms * phi0)
            spec[row, (L - ms[1:]) % L] = minus[1:] * np.exp(-1j * ms[1:] * phi0)
        want = L * np.fft.ifft(spec, axis=1)
        got = grid[[n + r, n - 1 - r]].cpu().numpy()
        errs.append(float(np.linalg.norm(got - want) / np.linalg.norm(want)))
    checks["synthesis_rows_vs_numpy_max"] = max(errs)
    del yb
    hgrid = grid.cpu().numpy()

    inv = run.inverse(grid)
    print(f"inverse: device {inv['device_ms']:.1f} ms (ALT {inv['alt_ms']:.1f} ms, "
          f"{inv['alt_gbs']:.0f} GB/s), plan {inv['plan_s']:.0f} s (replanned "
          f"{inv['replanned']} chunks)", file=sys.stderr, flush=True)
    back = inv.pop("coeffs")
    if args.oracle_all:
        bo = ora["back"]
        per = [float(np.linalg.norm(back[offs0[i]:offs0[i + 1]] - bo[offs0[i]:offs0[i + 1]])
                     / np.linalg.norm(bo[offs0[i]:offs0[i + 1]])) for i in range(len(offs0) - 1)]
        ora_res["inv_rel_l2"] = float(np.linalg.norm(back - bo) / np.linalg.norm(bo))
        ora_res["inv_worst_order"] = max(per)
        ora_res["inv_worst_order_m"] = int(np.argmax(per)) - (2 * n - 1)
        ora_res["oracle_seconds"] = ora["seconds"]
        ora_res["oracle"] = ("oracle/apply.py alt_forward / alt_inverse on every order's plan "
                             "(threads), numpy pocketfft for the phi stage; inverse input = "
                             "pocketfft spectrum of the GPU grid")
        checks["global_vs_oracle"] = ora_res
        ora["spectrum"] = ora["back"] = None
    if subset is None:
        checks["roundtrip_rel_l2"] = float(np.linalg.norm(back - flat) / np.linalg.norm(flat))
    else:
        sel = np.concatenate([np.arange(offs0[(2 * n - 1) + mm], offs0[(2 * n - 1) + mm + 1])
                              for m in subset for mm in ((m, -m) if m else (m,))])
        checks["roundtrip_rel_l2"] = float(np.linalg.norm(back[sel] - flat[sel])
                                           / np.linalg.norm(flat[sel]))
    # inverse of sampled orders from the GPU grid's spectrum columns (numpy
    # pocketfft, as the reference: sht.py:161)
    errs = []
    spec_all = np.fft.fft(hgrid, axis=1) / L
    for m in samples:
        for sgn in ((1,) if m == 0 else (1, -1)):
            mm = sgn * m
            b = mm % L
            col = spec_all[:, b] * np.exp(-1j * mm * phi0)
            with threadpool_limits(limits=1):
                t = time.perf_counter()
                want = OA.alt_inverse(plans[m], col)
                cpu["seconds"] += time.perf_counter() - t
            i = (2 * n - 1) + mm
            got = back[offs[i]:offs[i + 1]]
            errs.append(float(np.linalg.norm(got - want) / np.linalg.norm(want)))
        cpu["values"] += int(plans[m].stats["total_nnz"]) if hasattr(plans[m], "stats") \
            else 0
    del spec_all
    # (round 1 built this spectrum with a direct DFT sum whose phases
    # exp(-2 pi i b j / L) lose ~1e-11 at b*j ~ 2.7e8: that, not the GPU, was
    # the 2.9e-11 of r01_ooc_n4096.json).  The exact check below feeds the
    # oracle the GPU's own analysis output (weighted folds in the θ-major buffer)
    checks["alt_inverse_vs_oracle_pocketfft_spectrum_max"] = max(errs)
    errs = []
    for m in samples:
        p = plans[m]
        e = run.node_entries(m)
        for sgn, cols in ((1, (0, 1)), (-1, (2, 3))):
            if m == 0 and sgn < 0:
                continue
            want = np.zeros(2 * n - m, dtype=np.complex128)
            for par, spec, blocks, sl in ((0, p.spec_odd, p.blocks_odd, slice(1, None, 2)),
                                          (1, p.spec_even, p.blocks_even, slice(0, None, 2))):
                if spec is None:
                    continue
                re = OA.apply_half_transpose(blocks, e[par][:, cols[0]], spec.num_cols)
                im = OA.apply_half_transpose(blocks, e[par][:, cols[1]], spec.num_cols)
                want[sl] = re + 1j * im
            i = (2 * n - 1) + sgn * m
            got = back[offs[i]:offs[i + 1]]
            errs.append(float(np.linalg.norm(got - want) / np.linalg.norm(want)))
    checks["alt_inverse_vs_oracle_max"] = max(errs)

    real_inv = None
    if args.real_grid:
        # config 5's inverse input: a real grid, iid U(-1,1), promoted to
        # complex (sht.py:151-166)
        g = torch.from_numpy(np.random.default_rng(5).uniform(-1.0, 1.0, (2 * n, L))) \
            .to(torch.complex128).cuda()
        real_inv = run.inverse(g)
        rb = real_inv.pop("coeffs")
        errs = []
        for m in samples:
            p = plans[m]
            e = run.node_entries(m)
            for sgn, cols in ((1, (0, 1)), (-1, (2, 3))):
                if m == 0 and sgn < 0:
                    continue
                want = np.zeros(2 * n - m, dtype=np.complex128)
                for par, spec, blocks, sl in ((0, p.spec_odd, p.blocks_odd, slice(1, None, 2)),
                                              (1, p.spec_even, p.blocks_even, slice(0, None, 2))):
                    if spec is None:
                        continue
                    want[sl] = OA.apply_half_transpose(blocks, e[par][:, cols[0]], spec.num_cols) \
                        + 1j * OA.apply_half_transpose(blocks, e[par][:, cols[1]], spec.num_cols)
                i = (2 * n - 1) + sgn * m
                got = rb[offs[i]:offs[i + 1]]
                errs.append(float(np.linalg.norm(got - want) / np.linalg.norm(want)))
        checks["real_grid_alt_inverse_vs_oracle_max"] = max(errs)
        print(f"real-grid inverse: device {real_inv['device_ms']:.1f} ms", file=sys.stderr, flush=True)

    v_n = fwd["payload_values"]
    dev_ms = fwd["device_ms"] + inv["device_ms"]
    resident = [c for c in fwd["chunks"] if c.get("resident")]
    res = {
        "workload": f"C3: SHT fwd+inv N={n}, tol {args.tol:g}, one B200, orders in "
                    f"{len(run.chunks)} chunks (plan > HBM: planned/packed/uploaded per chunk)",
        "n": n, "grid": [2 * n, L], "chunks": len(run.chunks),
        "payload_values": v_n, "payload_gb": 8 * v_n / 1e9,
        "device_ms_fwd": fwd["device_ms"], "device_ms_inv": inv["device_ms"],
        "transforms_per_s_device": 1e3 / dev_ms,
        "alt_ms": [fwd["alt_ms"], inv["alt_ms"]],
        "alt_gbs": [fwd["alt_gbs"], inv["alt_gbs"]],
        "dft_ms": [fwd["dft_ms"], inv["dft_ms"]],
        "pack_copy_ms": [fwd["pack_ms"] + fwd["copy_ms"], inv["pack_ms"] + inv["copy_ms"]],
        "host_s": {"plan": [fwd["plan_s"], inv["plan_s"]],
                   "pack_upload": [fwd["pack_upload_s"], inv["pack_upload_s"]],
                   "replanned_chunks_inverse": inv["replanned"],
                   "total_wall": time.perf_counter() - t0},
        "checks": checks,
        "samples": samples,
        "alt_ms_per_chunk_fwd": fwd["alt_ms_per_chunk"],
        "regen": args.regen,
        "resident_chunks_after_forward": len(resident),
        "resident_tile_gb": sum(c.get("tile_gb", 0.0) for c in resident),
        "gpu_mem_used_gb_after_forward": fwd.get("gpu_mem_used_gb"),
    }
    if only is not None:
        res["workload"] = (f"C5-style sampled run: N={n}, tol {args.tol:g}, one B200, chunks {only} "
                           f"of {len(run.chunks)} ({len(subset)} orders, coefficients (1+k)^-"
                           f"{args.decay:g} on them, zero elsewhere) through the full "
                           f"{2 * n} x {L} grid and DFT stage")
        res["orders_processed"] = len(subset)
        res["note"] = ("device_ms / transforms_per_s cover the processed chunks' ALT plus the "
                       "full-grid DFT stage; not a whole-plan number")
    if real_inv is not None:
        res["real_grid_inverse_device_ms"] = real_inv["device_ms"]
        res["real_grid_inverse_dft_ms"] = real_inv["dft_ms"]
    if cpu["values"]:
        res["cpu_baseline"] = {
            "kind": "port", "cores": 1,
            "sample": f"oracle alt_forward+alt_inverse of orders {samples} (+m and -m), "
                      "1 core; extrapolated to all orders by payload values",
            "sample_seconds": cpu["seconds"],
            "extrapolated_fwd_inv_s": cpu["seconds"] * v_n / cpu["values"]}
    line = json.dumps(res)
    print(line)
    out = args.out.format(n=n)
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    with open(out, "w") as fh:
        fh.write(line + "\n")
    run.close()


if __name__ == "__main__":
    main()
