"""Transfer roofline for the inter-stage messages:
achieved GB/s of the P2P link mode's copy kernel (adaptra_p2p_copy, 32 CTAs)
GPU0 -> GPU1 over NVLink and within one GPU (HBM), for the message sizes of
C1 (8 MiB) and C2 (16 MiB) and larger, next to the copy engines
(torch copy_ / cudaMemcpyPeer) as context.  Peaks: NVLink 5 900 GB/s per
direction (B200_PROFILING.md), HBM from MEASURED_PEAKS.json (read + write
bytes).  Needs 2 GPUs: gpurun --gpus 2 -- python scripts/nvlink_bench.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2504_19232_b200 import _lib as L  # noqa: E402

lib = L.lib()
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peaks = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))
hbm_peak = peaks.get("hbm_gbs", 6542.7)
nvl_peak = 900.0
n_gpu = torch.cuda.device_count()
torch.cuda.set_device(0)


def timed(fn, stream, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = []
for mib in (8, 16, 64, 256):
    n = mib * 2**20
    src0 = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    dst0 = torch.empty(n, dtype=torch.uint8, device="cuda:0")
    st0 = torch.cuda.Stream(device=0)
    ms = timed(lambda: L.check(lib.adaptra_p2p_copy(dst0.data_ptr(), src0.data_ptr(), n, st0.cuda_stream)), st0)
    gbs = 2 * n / (ms / 1e3) / 1e9  # read + write
    out.append({"path": "HBM (same GPU), adaptra_p2p_copy", "MiB": mib, "us": round(ms * 1e3, 1),
                "GBps_rw": round(gbs, 1), "peak": hbm_peak, "frac": round(gbs / hbm_peak, 3)})
    if n_gpu >= 2:
        dst1 = torch.empty(n, dtype=torch.uint8, device="cuda:1")
        ms = timed(lambda: L.check(lib.adaptra_p2p_copy(dst1.data_ptr(), src0.data_ptr(), n, st0.cuda_stream)), st0)
        gbs = n / (ms / 1e3) / 1e9
        out.append({"path": "NVLink GPU0 -> GPU1, adaptra_p2p_copy (SM stores)", "MiB": mib, "us": round(ms * 1e3, 1),
                    "GBps": round(gbs, 1), "peak": nvl_peak, "frac": round(gbs / nvl_peak, 3)})
        ms = timed(lambda: dst1.copy_(src0, non_blocking=True), torch.cuda.current_stream(0))
        gbs = n / (ms / 1e3) / 1e9
        out.append({"path": "NVLink GPU0 -> GPU1, copy engine (torch copy_)", "MiB": mib, "us": round(ms * 1e3, 1),
                    "GBps": round(gbs, 1), "peak": nvl_peak, "frac": round(gbs / nvl_peak, 3)})
for r in out:
    print(json.dumps(r), flush=True)
