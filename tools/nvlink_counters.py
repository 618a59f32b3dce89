"""NVLink bytes per GPU around a command (GPU box): reads `nvidia-smi nvlink -gt d`
(per-link data Tx/Rx counters, KiB) before and after, prints per-GPU MB moved.
usage: python tools/nvlink_counters.py OUT.json -- <command ...>"""
import json
import re
import subprocess
import sys
import time


def counters():
    out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d"], capture_output=True, text=True).stdout
    gpu, res = None, {}
    for line in out.splitlines():
        m = re.match(r"GPU (\d+):", line.strip())
        if m:
            gpu = int(m.group(1))
            res[gpu] = {"tx_kib": 0, "rx_kib": 0}
            continue
        m = re.search(r"Data Tx:\s*(\d+)\s*KiB", line)
        if m and gpu is not None:
            res[gpu]["tx_kib"] += int(m.group(1))
        m = re.search(r"Data Rx:\s*(\d+)\s*KiB", line)
        if m and gpu is not None:
            res[gpu]["rx_kib"] += int(m.group(1))
    return res, out


if __name__ == "__main__":
    out_path = sys.argv[1]
    cmd = sys.argv[sys.argv.index("--") + 1:]
    a, raw_a = counters()
    t0 = time.time()
    rc = subprocess.run(cmd).returncode
    secs = time.time() - t0
    b, raw_b = counters()
    per = {g: {"tx_MB": round((b[g]["tx_kib"] - a[g]["tx_kib"]) * 1024 / 1e6, 1),
               "rx_MB": round((b[g]["rx_kib"] - a[g]["rx_kib"]) * 1024 / 1e6, 1)} for g in b if g in a}
    json.dump({"cmd": cmd, "rc": rc, "seconds": round(secs, 2), "per_gpu": per, "raw_before": raw_a[:4000]},
              open(out_path, "w"), indent=1)
    print(json.dumps(per))
    sys.exit(rc)
