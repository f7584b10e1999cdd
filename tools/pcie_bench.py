"""Host<->device copy bandwidth of this box (pinned memory), the bound of the e2e MatMult:
H2D alone, D2H alone, and both at once on two streams (PCIe is full duplex)."""
import json

import torch


def main(nbytes=134217728, reps=10):
    n = nbytes // 8
    h_in = torch.empty(n, dtype=torch.float64).pin_memory()
    h_out = torch.empty(n, dtype=torch.float64).pin_memory()
    d_a = torch.empty(n, dtype=torch.float64, device="cuda")
    d_b = torch.ones(n, dtype=torch.float64, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for name, ops in (("h2d", [(d_a, h_in, s1)]), ("d2h", [(h_out, d_b, s2)]),
                      ("both", [(d_a, h_in, s1), (h_out, d_b, s2)])):
        best = 1e9
        for _ in range(reps):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for dst, src, st in ops:
                st.wait_event(e0)
                with torch.cuda.stream(st):
                    dst.copy_(src, non_blocking=True)
            for _, _, st in ops:
                torch.cuda.current_stream().wait_stream(st)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) * 1e-3)
        res[name + "_GBps_per_direction"] = nbytes / best / 1e9
    # the e2e pipeline's pattern: 16 chunk uploads on one stream, 16 chunk downloads on another,
    # download k after upload k+1 (what the SpMV of chunk k needs), no kernels
    C = 16
    step = n // C
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        s1.wait_event(e0)
        s2.wait_event(e0)
        evs = []
        for k in range(C):
            with torch.cuda.stream(s1):
                d_a[k * step:(k + 1) * step].copy_(h_in[k * step:(k + 1) * step], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(s1)
                evs.append(ev)
        for k in range(C):
            s2.wait_event(evs[min(k + 1, C - 1)])
            with torch.cuda.stream(s2):
                h_out[k * step:(k + 1) * step].copy_(d_b[k * step:(k + 1) * step], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s2)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) * 1e-3)
    res["pipeline16_ms"] = best * 1e3
    print(json.dumps({"bench": "pcie", "bytes": nbytes, **res}))


if __name__ == "__main__":
    main()
