"""Summarise an `ncu --set full` report of one bench step (dev tool).

  python tools/ncu_summary.py gpurun_out/prof_mix.ncu-rep profiles/r01_ncu_full_n1_mixtral_s2.txt \
      [--traffic profiles/gemm_traffic_mixtral.json --flops-per-step F --header "..."]

Writes one line per launch (kernel | ms | SM clock | tensor-pipe active % | L2 hit % |
DRAM read / write GB | grid | block | regs | dyn smem) and, with --traffic, the mean
DRAM bytes per grouped-GEMM launch that bench.py reports as roofline.traffic.
"""
import argparse
import csv
import io
import json
import subprocess

COLS = [
    ("gpu__time_duration.sum", "ms"),
    ("sm__cycles_elapsed.avg.per_second", "SM GHz"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor %"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("dram__bytes_read.sum", "DRAM rd GB"),
    ("dram__bytes_write.sum", "DRAM wr GB"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem KB"),
]
NAMES = {
    "grouped_gemm_pair_kernel<0, 0, 0, 1>": "fwd gate-up + SwiGLU",
    "grouped_gemm_pair_kernel<0, 0, 0, 0>": "fwd down (+ y row scatter)",
    "grouped_gemm_pair_kernel<0, 1, 0, 2>": "bwd down-dgrad + SwiGLU'",
    "grouped_gemm_pair_kernel<0, 1, 0, 0>": "bwd up-dgrad dX (+ row scatter)",
    "grouped_gemm_pair_kernel<1, 1, 1, 3>": "wgrad (K-grouped, fp32)",
}


def to_gb(v, unit):
    return v / {"byte": 1e9, "Kbyte": 1e6, "Mbyte": 1e3, "Gbyte": 1.0}.get(unit, 1.0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--traffic")
    ap.add_argument("--header", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    name_i = hdr.index("Kernel Name")
    lines, gemm_bytes, gemm_pipe = [], [], []
    for r in data:
        full = r[name_i]
        short = full.split("(")[0].replace("void ", "").replace("fsep::", "").replace("(anonymous namespace)::", "")
        key = next((k for k in NAMES if k in full.replace("(bool)", "").replace("(int)", "")), None)
        label = f"{short} {NAMES[key]}" if key else short
        vals = []
        rd = wr = 0.0
        for c, _ in COLS:
            if c not in hdr:
                vals.append("n/a")
                continue
            i = hdr.index(c)
            v = r[i].replace(",", "")
            try:
                f = float(v)
            except ValueError:
                vals.append(v)
                continue
            if c.startswith("dram__bytes"):
                f = to_gb(f, units[i])
                rd, wr = (f, wr) if "read" in c else (rd, f)
            vals.append(f"{f:.4g}")
        if "grouped_gemm_pair_kernel" in full:
            gemm_bytes.append((rd + wr) * 1e9)
            try:
                gemm_pipe.append((float(vals[0]), float(vals[2])))  # (ms, tensor-pipe %)
            except ValueError:
                pass
        lines.append(" | ".join([label] + vals))
    with open(a.out, "w") as f:
        if a.header:
            f.write("".join(f"# {h}\n" for h in a.header.split("\\n")))
        f.write("# kernel | " + " | ".join(n for _, n in COLS) + "\n")
        f.write("\n".join(lines) + "\n")
    if a.traffic and gemm_bytes:
        tot = sum(ms for ms, _ in gemm_pipe)
        pipe = sum(ms * pct for ms, pct in gemm_pipe) / tot if tot else None
        json.dump({"dram_bytes_per_launch": sum(gemm_bytes) / len(gemm_bytes), "launches_averaged": len(gemm_bytes),
                   "tensor_pipe_active_pct": round(pipe, 2) if pipe is not None else None,
                   "source": a.out,
                   "note": "mean dram__bytes_read.sum + dram__bytes_write.sum over the CTA-pair grouped-GEMM launches "
                           "of one bench step (ncu --set full --clock-control none); tensor_pipe_active_pct: "
                           "sm__pipe_tensor_cycles_active (pct of peak, elapsed) weighted by launch time"},
                  open(a.traffic, "w"), indent=1)
    print(f"{len(lines)} launches, {len(gemm_bytes)} pair-GEMM launches")


if __name__ == "__main__":
    main()
