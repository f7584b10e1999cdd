"""SF-pingpong / SF-unpack microbenchmark on NVLink 5 (the paper's Listing 5).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/sf_bench.py [--graph]
    (SPMAT_SF=nccl: the NCCL transport; --graph: replay the iterations from a CUDA graph, so
    the numbers are device time rather than the Python launch rate)

Two ranks; rank 0 owns n consecutive roots, rank 1 has n leaves connected one-on-one in order
(the right SF of the paper's Fig. 1).  One iteration = SFBcastBegin/End then
SFReduceBegin/End with op REPLACE (pingpong: user buffers are the transport buffers) or SUM
(unpack: an add kernel on the receiving side).  Reported: one-way latency = iteration time / 2,
measured with CUDA events on the caller's stream (max over ranks), and the bandwidth n*8 B /
one-way time.  Unlike GPU-aware MPI there is no device synchronisation before sending: the
whole iteration is stream-ordered.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_08646_b200 as sp  # noqa: E402
from paper_2406_08646_b200 import dist as sd  # noqa: E402


def main():
    P, r = int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("RANK", 0))
    assert P == 2, "SF-pingpong uses two ranks"
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
    comm = sp.Comm(device=local, nranks=P, rank=r)
    graph = "--graph" in sys.argv
    transport = None
    stream = torch.cuda.current_stream()
    rows = []
    for logn in range(0, 24, 2):  # 8 B .. 32 MB
        n = 1 << logn
        nroots = n if r == 0 else 0
        if r == 1:
            sf = sp.StarForest(comm, 0, None, [0] * n, list(range(n)))
        else:
            sf = sp.StarForest(comm, nroots, None, [], [])
        rdata = torch.arange(max(nroots, 1), dtype=torch.float64, device="cuda")
        ldata = torch.zeros(max(n if r == 1 else 0, 1), dtype=torch.float64, device="cuda")
        res = {"n": n, "bytes": 8 * n}
        transport = {2: "flagged lines over NVLink peer memory", 1: "NCCL p2p over NVLink 5"}.get(sf.transport())
        for name, op in (("replace", sp.REPLACE), ("sum", sp.SUM)):
            niter = 200 if n <= (1 << 16) else 50

            def iteration(st):
                sf.bcast_begin(rdata, ldata, op, st)
                sf.bcast_end(rdata, ldata, op, st)
                sf.reduce_begin(ldata, rdata, op, st)
                sf.reduce_end(ldata, rdata, op, st)

            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            for _ in range(10):
                iteration(stream)
            if graph:  # device time: the iterations replayed from a CUDA graph
                g, gs = torch.cuda.CUDAGraph(), torch.cuda.Stream()
                gs.wait_stream(stream)
                with torch.cuda.graph(g, stream=gs):
                    for _ in range(niter):
                        iteration(gs)
                torch.cuda.synchronize()
                sd.barrier()
                e0.record(stream)
                g.replay()
            else:
                torch.cuda.synchronize()
                sd.barrier()
                e0.record(stream)
                for _ in range(niter):
                    iteration(stream)
            e1.record(stream)
            torch.cuda.synchronize()
            us = sd.max_over_ranks(e0.elapsed_time(e1) * 1e3 / niter / 2)
            res[f"{name}_us"] = us
            res[f"{name}_GBps"] = 8 * n / us / 1e3
            if "--breakdown" in sys.argv and n >= (1 << 18) and name == "replace":
                # per-call device time of each half on each rank (eager, events between calls):
                # rank 0's bcast_begin = the put kernel (stores over NVLink), rank 1's
                # bcast_end = the consuming kernel (waits for the lines, copies them out)
                ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
                acc = [0.0] * 4
                for _ in range(niter):
                    sd.barrier()
                    torch.cuda.synchronize()
                    ev[0].record(stream)
                    sf.bcast_begin(rdata, ldata, op, stream)
                    ev[1].record(stream)
                    sf.bcast_end(rdata, ldata, op, stream)
                    ev[2].record(stream)
                    sf.reduce_begin(ldata, rdata, op, stream)
                    ev[3].record(stream)
                    sf.reduce_end(ldata, rdata, op, stream)
                    ev[4].record(stream)
                    torch.cuda.synchronize()
                    for k in range(4):
                        acc[k] += ev[k].elapsed_time(ev[k + 1]) * 1e3 / niter
                allp = [None, None]
                torch.distributed.all_gather_object(allp, acc)
                res["breakdown_us"] = {"rank0_bcast_begin(put)": allp[0][0], "rank1_bcast_end(take)": allp[1][1],
                                       "rank1_reduce_begin(put)": allp[1][2], "rank0_reduce_end(take)": allp[0][3]}
                res["put_GBps"] = 8 * n / allp[0][0] / 1e3 if allp[0][0] > 0 else None
        rows.append(res)
        sf.close()
    if r == 0:
        print(json.dumps({"bench": "sf_pingpong", "transport": transport,
                          "timing": "CUDA graph replay" if graph else "eager launches", "rows": rows}),
              flush=True)
        print(f"{'bytes':>10s} {'REPLACE us':>11s} {'GB/s':>8s} {'SUM us':>9s} {'GB/s':>8s}")
        for x in rows:
            print(f"{x['bytes']:10d} {x['replace_us']:11.2f} {x['replace_GBps']:8.2f} "
                  f"{x['sum_us']:9.2f} {x['sum_GBps']:8.2f}")
    comm.close()
    torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
