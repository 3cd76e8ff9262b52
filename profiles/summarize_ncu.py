"""Summarize an ncu --set full capture of the FFT pass kernels into profiles/.

    python profiles/summarize_ncu.py gpurun_out/prof_c3_v8.ncu-rep c3 profiles/r01/ncu_full_c3_v8.md [traffic.json]

Writes a markdown table of the metrics the roofline uses and updates
profiles/ncu_traffic.json ({config: {pass index: dram bytes read+write}})
which bench.py reports as roofline.traffic.
"""
import csv
import json
import subprocess
import sys
from pathlib import Path

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "LSU data pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "registers"),
    ("launch__block_size", "block"),
    ("launch__grid_size", "grid"),
    ("smsp__inst_executed.sum", "warp instructions"),
]
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}


def main(rep, config, out_md, traffic_json=None):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# ncu --set full, {config}: FFT pass kernels of one solve ({Path(rep).name})", "",
             "| metric | " + " | ".join(f"pass {i}" for i in range(len(data))) + " |",
             "|---|" + "---|" * len(data)]
    for key, name in METRICS:
        if key not in idx:
            continue
        u = units[idx[key]]
        lines.append(f"| {name} ({u}) | " + " | ".join(r[idx[key]] for r in data) + " |")
    names = [r[idx["Kernel Name"]][:60] for r in data]
    lines += ["", "kernels: " + "; ".join(f"{i}: {n}" for i, n in enumerate(names))]
    Path(out_md).write_text("\n".join(lines) + "\n")
    traffic_path = Path(traffic_json) if traffic_json else Path(__file__).resolve().parent / "ncu_traffic.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    per = {}
    for i, r in enumerate(data):
        rd = float(r[idx["dram__bytes_read.sum"]]) * SCALE[units[idx["dram__bytes_read.sum"]]]
        wr = float(r[idx["dram__bytes_write.sum"]]) * SCALE[units[idx["dram__bytes_write.sum"]]]
        per[str(i)] = rd + wr if rd + wr == rd + wr else None   # NaN (metric not collected) -> null
    traffic[config] = per
    traffic_path.write_text(json.dumps(traffic, indent=1) + "\n")
    print(Path(out_md).read_text())


if __name__ == "__main__":
    main(*sys.argv[1:5])
