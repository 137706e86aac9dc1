"""Summarise ncu reports (run here, on the CPU box) into profiles/.

  python scripts/ncu_summary.py <tag> gpurun_out/prof_combine.ncu-rep [...]

Writes profiles/<tag>_<name>.txt (key metrics) and updates
profiles/ncu_traffic.json (dram bytes per launch per kernel class, read by
bench.py for roofline.traffic).
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct"]
CLASS = {"OpCombine": "combine", "OpMask": "mask", "k_mac_sigma": "sigma", "OpOpen": "open",
         "k_matrix_combine": "linear_combine", "k_modgemm": "gemm"}


def raw(rep):
    out = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def main():
    tag = sys.argv[1]
    prof = ROOT / "profiles"
    prof.mkdir(exist_ok=True)
    tj = prof / "ncu_traffic.json"
    traffic = json.loads(tj.read_text()) if tj.exists() else {}
    for rep in sys.argv[2:]:
        kernels, units = raw(rep)
        lines = []
        for k in kernels:
            name = k.get("Kernel Name", "?")
            cls = next((v for key, v in CLASS.items() if key in name), "other")
            lines.append(f"kernel: {name[:160]}")
            for key in KEYS:
                if key in k:
                    lines.append(f"  {key} = {k[key]} {units.get(key, '')}")

            def to_bytes(key):
                v = float(k[key].replace(",", ""))
                u = units.get(key, "byte").lower()
                return v * {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9}.get(u, 1)

            if "dram__bytes_read.sum" in k:
                traffic[cls] = {"dram_bytes_per_launch": int(to_bytes("dram__bytes_read.sum") +
                                                             to_bytes("dram__bytes_write.sum")),
                                "duration_us_under_ncu": k.get("gpu__time_duration.sum"), "report": Path(rep).name,
                                "tag": tag}
        out = prof / f"{tag}_{Path(rep).stem}.txt"
        out.write_text("\n".join(lines) + "\n")
        print(out)
    tj.write_text(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    main()
