"""Probe the NVML NVLink counters bench.py reads (run on the GPU box)."""
import pynvml as n
n.nvmlInit()
h = n.nvmlDeviceGetHandleByIndex(0)
links = []
for l in range(18):
    try:
        st = n.nvmlDeviceGetNvLinkState(h, l)
        links.append((l, st))
    except Exception as e:
        links.append((l, repr(e)))
print("links", links)
for fid in (138, 139, 202, 204):
    try:
        v = n.nvmlDeviceGetFieldValues(h, [(fid, 0)])
        print(fid, v[0].nvmlReturn, v[0].valueType, v[0].value.ullVal)
    except Exception as e:
        print(fid, "err", repr(e))
    try:
        v = n.nvmlDeviceGetFieldValues(h, [fid])
        print(fid, "noscope", v[0].nvmlReturn, v[0].valueType, v[0].value.ullVal)
    except Exception as e:
        print(fid, "noscope err", repr(e))
