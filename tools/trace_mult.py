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
    G, nitems = int(t[-2]), int(t[-1])  # header: CTAs, off-diagonal work items
    cta = t[:4 * G].reshape(G, 4).astype(np.float64)
    # item record: start, compute start (boundary blocks written), end, (same as [1])
    items = t[4 * G:4 * G + 4 * nitems].reshape(nitems, 4).astype(np.float64) if nitems else np.zeros((0, 4))
    t0 = cta[:, 0].min()
    span = cta[:, 3].max() - t0
    term = cta[:, 2] - t0
    msg = [f"rank {r}: kernel span {span / 1e3:.1f} us, CTAs {G}, mode {A.halo_mode()}; per call "
           f"{per:.1f} us, call duration median {np.median(dur):.1f} us",
           f"  CTA start spread {np.ptp(cta[:, 0]) / 1e3:.1f} us; last-block done: min {term.min() / 1e3:.1f} "
           f"median {np.median(term) / 1e3:.1f} max {term.max() / 1e3:.1f} us; end max {(cta[:, 3].max() - t0) / 1e3:.1f}"]
    put = cta[:, 1][cta[:, 1] > 0] - t0
    if put.size:
        msg.append(f"  puts out: {put.size} CTAs, {put.min() / 1e3:.1f}..{put.max() / 1e3:.1f} us; "
                   f"kernel start (globaltimer) {int(t0) % 10**9 / 1e3:.1f} us")
    if nitems:
        st = items[:, 0] - t0
        wait = items[:, 1] - items[:, 0]
        comp = items[:, 2] - items[:, 1]
        msg.append(f"  items {nitems}: start {st.min() / 1e3:.1f}..{st.max() / 1e3:.1f} us; boundary-block "
                   f"wait median {np.median(wait) / 1e3:.2f} max {wait.max() / 1e3:.2f} us; ghost wait + "
                   f"compute median {np.median(comp) / 1e3:.2f} max {comp.max() / 1e3:.2f} us")
    for k in range(P):
        sd.barrier()
        if k == r:
            print("\n".join(msg), flush=True)
    A.close()
    comm.close()


if __name__ == "__main__":
    main()
