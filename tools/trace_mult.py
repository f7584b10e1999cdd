"""Device trace of the fused MatMult kernel (SPMAT_TRACE=1), one line of statistics per rank.

    SPMAT_TRACE=1 torchrun --nproc-per-node 2 tools/trace_mult.py [--config c4] [--at 0.5]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_08646_b200 as sp  # noqa: E402
import synth  # noqa: E402
from paper_2406_08646_b200 import dist as sd  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--graph", action="store_true",
                    help="replay the calls from a CUDA graph (no host launch gaps, ranks in lockstep)")
    a = ap.parse_args()
    P, r = int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("RANK", 0))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if P > 1:
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = sp.Comm(device=local, nranks=P, rank=r)
    if a.config in ("kuu", "bump"):  # the CG-benchmark problems (tools/cg_bench.py)
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from cg_bench import problem
        i, j, v, sizes = problem(a.config, P, r)
    else:
        i, j, v, sizes = synth.config_rank_coo(a.config, P, r, values="real", device="cuda")
    off = synth.offsets_from_sizes(sizes)
    A = sp.Mat(comm, sizes[r], sizes[r], off[-1], off[-1], i, j)
    A.set_values(v)
    del i, j, v
    x = synth.x_vector(off[r], off[r + 1], "real", device="cuda")
    y = torch.empty(sizes[r], dtype=torch.float64, device="cuda")
    for _ in range(a.reps):
        A.mult(x, y)
    torch.cuda.synchronize()
    # per-call device time with events around every call (launch gaps show as e[k+1]-e[k] > d)
    ev = [torch.cuda.Event(enable_timing=True, external=a.graph) for _ in range(2 * a.reps)]
    if a.graph:
        g, gs = torch.cuda.CUDAGraph(), torch.cuda.Stream()
        with torch.cuda.graph(g, stream=gs):
            for k in range(a.reps):
                ev[2 * k].record(gs)
                A.mult(x, y, gs)
                ev[2 * k + 1].record(gs)
        torch.cuda.synchronize()
        sd.barrier()
        g.replay()
    else:
        for k in range(a.reps):
            ev[2 * k].record()
            A.mult(x, y)
            ev[2 * k + 1].record()
    torch.cuda.synchronize()
    dur = [ev[2 * k].elapsed_time(ev[2 * k + 1]) * 1e3 for k in range(a.reps)]
    per = ev[0].elapsed_time(ev[-1]) * 1e3 / a.reps
    t = sp.spmat_trace_read(A.h)
    G, K = int(t[-2]), int(t[-1])  # header: CTAs, stamps per CTA
    # per CTA: consumer start, puts out, last block done, consumer end, comm warp saw the
    # boundary blocks, comm warp off-diagonal chunks done (0 = not recorded)
    cta = t[:K * G].reshape(G, K).astype(np.float64)
    t0 = cta[:, 0].min()
    end = max(cta[:, 3].max(), cta[:, 5].max())
    span = end - t0
    term = cta[:, 2] - t0
    msg = [f"rank {r}: kernel span {span / 1e3:.1f} us, CTAs {G}, mode {A.halo_mode()}; per call "
           f"{per:.1f} us, call duration median {np.median(dur):.1f} us",
           f"  CTA start spread {np.ptp(cta[:, 0]) / 1e3:.1f} us; last-block done: min {term.min() / 1e3:.1f} "
           f"median {np.median(term) / 1e3:.1f} max {term.max() / 1e3:.1f} us; consumers end max "
           f"{(cta[:, 3].max() - t0) / 1e3:.1f}"]
    put = cta[:, 1][cta[:, 1] > 0] - t0
    if put.size and A.halo_mode() == 2:
        msg.append(f"  puts out: {put.min() / 1e3:.1f}..{put.max() / 1e3:.1f} us")
    seen = cta[:, 4][cta[:, 4] > 0] - t0
    done = cta[:, 5][cta[:, 5] > 0] - t0
    if done.size:
        msg.append(f"  off-diagonal (comm warps): boundary blocks seen {seen.min() / 1e3:.1f}..{seen.max() / 1e3:.1f} us; "
                   f"chunks done median {np.median(done) / 1e3:.1f} max {done.max() / 1e3:.1f} us")
    for k in range(P):
        sd.barrier()
        if k == r:
            print("\n".join(msg), flush=True)
    A.close()
    comm.close()


if __name__ == "__main__":
    main()
