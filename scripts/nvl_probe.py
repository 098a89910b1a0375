"""Which NVLink byte counters does this driver expose? (NVML field values, per link and aggregate)."""
import pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
names = [n for n in dir(nv) if n.startswith("NVML_FI_DEV_NVLINK") and ("BYTES" in n or "THROUGHPUT" in n or "COUNT_X" in n or "COUNT_R" in n)]
for n in sorted(names):
    fid = getattr(nv, n)
    res = []
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            v = nv.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            res.append((scope, v.nvmlReturn, int(v.value.ullVal)))
        except Exception as e:
            res.append((scope, str(e)[:40]))
    print(n, fid, res)
try:
    print("link0 util ctrl", nv.nvmlDeviceGetNvLinkUtilizationCounter(h, 0, 0))
except Exception as e:
    print("util counter:", e)
