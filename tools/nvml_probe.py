"""NVLink data bytes per GPU from NVML throughput counters (TX/RX, summed
over links); prints one JSON line {gpu: {"tx": bytes, "rx": bytes}}.  Used
around a multi-GPU bench run to get the NVLink bytes of its steps."""
import json

import pynvml as N

N.nvmlInit()
out = {}
for i in range(N.nvmlDeviceGetCount()):
    h = N.nvmlDeviceGetHandleByIndex(i)
    rec = {}
    for key, fid in (("tx", N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX),
                     ("rx", N.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX)):
        tot, how = 0, None
        for scope in range(18):                      # per link
            try:
                r = N.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            except Exception as e:  # noqa: BLE001
                how = f"err {e}"
                break
            if r.nvmlReturn != 0:
                continue
            tot += int(r.value.ullVal)
            how = "per-link"
        if how is None or how.startswith("err"):
            try:
                r = N.nvmlDeviceGetFieldValues(h, [fid])[0]
                if r.nvmlReturn == 0:
                    tot, how = int(r.value.ullVal), "device"
            except Exception as e:  # noqa: BLE001
                how = f"err {e}"
        rec[key] = tot
        rec[key + "_how"] = how
    out[i] = rec
print(json.dumps(out))
