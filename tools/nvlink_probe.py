"""Probe (tools/): which NVLink byte counters this box exposes (NVML field values per link,
nvidia-smi nvlink -gt d)."""
import subprocess

import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
for name in ("NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX",
             "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX"):
    fid = getattr(pynvml, name)
    for scope in (0, 1, 0xFFFFFFFF):
        try:
            v = pynvml.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            print(name, hex(scope), "ret", v.nvmlReturn, "val", v.value.ullVal)
        except Exception as e:  # noqa: BLE001
            print(name, scope, "exc", e)
for args in (["nvidia-smi", "nvlink", "-gt", "d", "-i", "0"], ["nvidia-smi", "nvlink", "-s", "-i", "0"]):
    r = subprocess.run(args, capture_output=True, text=True)
    print(" ".join(args), "rc", r.returncode)
    print(r.stdout[:1500], r.stderr[:300])
