"""NVLink ceilings of this box (2 GPUs, one process): copy-engine peer copies of 1 MB..1 GB
(cudaMemcpyPeerAsync via torch), and NVML's NVLink byte counters around them -- the reference
points for the halo and SF-pingpong numbers (context for profiles/r02_nvlink.md)."""
import json
import sys
import time

import torch

try:
    import pynvml as nv
    nv.nvmlInit()
except Exception:  # noqa: BLE001
    nv = None

FIELDS = {"count_xmit_bytes": 202, "count_rcv_bytes": 204, "thr_data_tx_kib": 138, "thr_data_rx_kib": 139}


def counters(h):
    out = {}
    if nv is None:
        return out
    for name, fid in FIELDS.items():
        tot, ok, rets = 0, 0, set()
        for link in list(range(18)) + [0xFFFFFFFF]:
            try:
                v = nv.nvmlDeviceGetFieldValues(h, [(fid, link)])[0]
                rets.add(int(v.nvmlReturn))
                if v.nvmlReturn == 0:
                    tot += int(v.value.ullVal)
                    ok += 1
            except Exception as ex:  # noqa: BLE001
                rets.add(type(ex).__name__)
        out[name] = (tot, ok)
        RETS[name] = sorted(map(str, rets))
    return out


RETS = {}


def main():
    assert torch.cuda.device_count() >= 2
    h0 = nv.nvmlDeviceGetHandleByIndex(0) if nv else None
    rows = []
    for mb in (1, 8, 32, 128, 1024):
        n = mb * (1 << 20) // 8
        a = torch.randn(n, dtype=torch.float64, device="cuda:0")
        b = torch.empty(n, dtype=torch.float64, device="cuda:1")
        for _ in range(3):
            b.copy_(a)
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        it = 20
        c0 = counters(h0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.device(0):
            e0.record()
            for _ in range(it):
                b.copy_(a)
            e1.record()
        torch.cuda.synchronize(0)
        torch.cuda.synchronize(1)
        time.sleep(0.2)
        c1 = counters(h0)
        ms = e0.elapsed_time(e1) / it
        d = {k: (c1[k][0] - c0[k][0], c1[k][1]) for k in c1}
        rows.append({"MB": mb, "us": ms * 1e3, "GBps": mb * (1 << 20) / ms / 1e6,
                     "counter_delta_per_copy": {k: v[0] / it for k, v in d.items()},
                     "links_answering": {k: v[1] for k, v in d.items()}})
        rows[-1]["nvml_returns"] = dict(RETS)
        print(json.dumps(rows[-1]), flush=True)
    print(json.dumps({"bench": "nvlink_ce_copy", "rows": rows}))


if __name__ == "__main__":
    sys.exit(main())
