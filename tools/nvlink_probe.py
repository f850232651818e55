"""Validate the NVML NVLink byte counters used by bench.py: read them around a
known peer copy (1 GiB GPU0 -> GPU1) and print the deltas per field."""
import sys
import time

import pynvml as N
import torch

FIELDS = {"THROUGHPUT_DATA_TX": N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX,
          "THROUGHPUT_DATA_RX": N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX,
          "THROUGHPUT_RAW_TX": N.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX,
          "THROUGHPUT_RAW_RX": N.NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX,
          "COUNT_XMIT_BYTES": N.NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES,
          "COUNT_RCV_BYTES": N.NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES}


def read(h):
    out = {}
    for name, fid in FIELDS.items():
        try:
            vals = N.nvmlDeviceGetFieldValues(h, [(fid, 0xFFFFFFFF)])
            v = vals[0]
            out[name] = (v.nvmlReturn, v.value.ullVal)
        except Exception as e:
            out[name] = ("exc", str(e)[:60])
    return out


N.nvmlInit()
hs = [N.nvmlDeviceGetHandleByIndex(i) for i in range(torch.cuda.device_count())]
a = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:0")
b = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:1")
b.copy_(a)
torch.cuda.synchronize(0); torch.cuda.synchronize(1)
time.sleep(0.2)
before = [read(h) for h in hs[:2]]
for _ in range(4):
    b.copy_(a)
torch.cuda.synchronize(0); torch.cuda.synchronize(1)
time.sleep(0.5)
after = [read(h) for h in hs[:2]]
for g in range(2):
    for name in FIELDS:
        r0, v0 = before[g][name]
        r1, v1 = after[g][name]
        d = (v1 - v0) if isinstance(v0, int) and isinstance(v1, int) else None
        print(f"gpu{g} {name:20s} rc {r0},{r1} delta {d}  (4 GiB copied GPU0->GPU1; ratio {d / (4 << 30) if d else None})")
