"""Summarise an ncu --set full report of one kernel into a markdown block and the
per-launch DRAM traffic json read by bench.py.

usage: python tools/ncu_summary.py REP.ncu-rep --freqs F --out profiles/NAME [--traffic-json path]"""
import argparse
import csv
import io
import json
import subprocess

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA inst issued % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 (DFMA) pipe active %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % (occupancy)"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__occupancy_limit_shared_mem", "CTAs/SM (smem limit)"),
]

UNIT = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--freqs", type=int, required=True, help="frequencies processed by the profiled launch")
    ap.add_argument("--out", required=True)
    ap.add_argument("--title", default="")
    ap.add_argument("--traffic-json", default=None)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    kname = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
    got = {}
    lines = [f"## {a.title or kname}", "", f"kernel: `{kname}`, frequencies in the launch: {a.freqs}", "",
             "| metric | value | unit |", "|---|---|---|"]
    for m, label in METRICS:
        if m in h:
            i = h.index(m)
            got[m] = (v[i], u[i])
            lines.append(f"| {label} (`{m}`) | {v[i]} | {u[i]} |")
    rd = float(got["dram__bytes_read.sum"][0].replace(",", "")) * UNIT.get(got["dram__bytes_read.sum"][1], 1)
    wr = float(got["dram__bytes_write.sum"][0].replace(",", "")) * UNIT.get(got["dram__bytes_write.sum"][1], 1)
    per = (rd + wr) / a.freqs
    lines += ["", f"DRAM traffic per frequency: {per / 1e6:.1f} MB (read {rd / a.freqs / 1e6:.1f} + "
              f"write {wr / a.freqs / 1e6:.1f})", ""]
    open(a.out + ".md", "w").write("\n".join(lines) + "\n")
    if a.traffic_json:
        json.dump({"dram_bytes_per_freq": per, "source": a.rep.split("/")[-1], "kernel": kname,
                   "freqs_in_profiled_launch": a.freqs}, open(a.traffic_json, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
