"""CGAsync-analogue timing: microseconds per CG iteration (one MatMult, two dots, three
vector updates, all scalars on the device, no host synchronisation), max over ranks.

    python tools/cg_bench.py [--config c4] [--iters 50]
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/cg_bench.py

Context: 690 us (CG) vs 676 us (CGAsync) per iteration on Bump_2911
(~3 M rows, 128 M nnz, 6 x V100); 300 vs 250 us on Kuu (~7 K rows, 340 K nnz).  The
"kuu" config here is a synthetic of that size (3-dof 27-point on 13^3 nodes: 6.6 K rows,
~0.5 M nnz); "bump" has Bump_2911's size AND density (synth config "bump": a 45-point 5x3x3
box stencil on 144^3 nodes, 2.99 M rows, 132 M nonzeros, 44 per row); "bump7" is round 1's
7-point 144^3 stand-in (same rows, 1/6 of the nonzeros).
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_08646_b200 as sp  # noqa: E402
import synth  # noqa: E402
from paper_2406_08646_b200 import dist as sd  # noqa: E402


def problem(name, P, r):
    if name == "kuu":
        n = 13
        sizes = synth.split_sizes(3 * n ** 3, P)
        off = synth.offsets_from_sizes(sizes)
        i, j, v = synth.elasticity_coo(n, values="int", device="cuda")
        keep = (i >= off[r]) & (i < off[r + 1])
        return i[keep], j[keep], v[keep], sizes
    if name == "bump7":  # round-1 stand-in: the row count of Bump_2911, not its density
        shape = (144, 144, 144)
        sizes = synth.split_sizes(144 ** 3, P)
        off = synth.offsets_from_sizes(sizes)
        i, j, v = synth.stencil_coo(shape, 7, rows=(off[r], off[r + 1]), values="int", device="cuda")
        return i, j, v, sizes
    i, j, v, sizes = synth.config_rank_coo(name, P, r, values="int", device="cuda")
    return i, j, v, sizes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="kuu,bump,c4")
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--breakdown", action="store_true",
                    help="also time MatMult alone and the dot alone (us per call)")
    a = ap.parse_args()
    P, r = int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if P > 1:
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = sp.Comm(device=local, nranks=P, rank=r)
    out = []
    for name in a.configs.split(","):
        i, j, v, sizes = problem(name, P, r)
        off = synth.offsets_from_sizes(sizes)
        M = off[-1]
        A = sp.Mat(comm, sizes[r], sizes[r], M, M, i, j)
        A.set_values(v)
        b = synth.x_vector(off[r], off[r + 1], "real", seed=1, device="cuda")
        x = torch.zeros(sizes[r], dtype=torch.float64, device="cuda")
        s = torch.cuda.current_stream()
        A.cg(b, x, 5, None, s)  # warm-up (allocates the workspace)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sd.barrier()
        e0.record(s)
        A.cg(b, x, a.iters, None, s)
        e1.record(s)
        torch.cuda.synchronize()
        us = sd.max_over_ranks(e0.elapsed_time(e1) * 1e3 / a.iters)
        parts = {}
        if a.breakdown:
            y = torch.empty_like(x)
            res = torch.empty(1, dtype=torch.float64, device="cuda")
            def fn_s(key, st):
                if key == "mult":
                    A.mult(b, y, st)
                else:
                    A.dot(b, x, res, st)

            for key in ("mult", "dot"):
                fn = lambda: fn_s(key, s)  # noqa: E731
                for _ in range(5):
                    fn()
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()  # device time, not the Python launch rate
                gs = torch.cuda.Stream()
                with torch.cuda.graph(g, stream=gs):
                    with torch.cuda.stream(gs):
                        for _ in range(a.iters):
                            fn_s(key, gs)
                torch.cuda.synchronize()
                sd.barrier()
                e0.record(s)
                g.replay()
                e1.record(s)
                torch.cuda.synchronize()
                parts[key] = sd.max_over_ranks(e0.elapsed_time(e1) * 1e3 / a.iters)
        nnz = sd.sum_over_ranks(A.info()["nnz_d"] + A.info()["nnz_o"])
        out.append({"config": name, "rows": M, "nnz": nnz, "P": P, "us_per_iteration": us,
                    "halo_mode": A.halo_mode(), **{f"us_{k}": v for k, v in parts.items()}})
        A.close()
    if r == 0:
        print(json.dumps({"bench": "cg_async", "rows": out}), flush=True)
        for o in out:
            print(f"{o['config']:6s} P={o['P']} rows={o['rows']:>10d} nnz={o['nnz']:>11d} "
                  f"{o['us_per_iteration']:9.1f} us/iteration"
                  + "".join(f"  {k[3:]} {o[k]:.1f}" for k in o if k.startswith("us_") and k != "us_per_iteration"))
    comm.close()
    if P > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
