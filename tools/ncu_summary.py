"""Summarise an ncu report (``--set full``) into the per-kernel JSON kept under profiles/.

python tools/ncu_summary.py REPORT.ncu-rep > profiles/<round>_ncu_full_summary.json
"""
import csv
import io
import json
import subprocess
import sys

FIELDS = {
    "duration_us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_read_per_s": "dram__bytes_read.sum.per_second",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread",
    "smem_per_block": "launch__shared_mem_per_block",
    "grid": "launch__grid_size",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
}


def main(path: str) -> None:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in data:
        e = {"kernel": r[col["Kernel Name"]][:60]}
        for k, m in FIELDS.items():
            if m in col:
                e[k] = f"{r[col[m]]} {units[col[m]]}".strip()
        res.append(e)
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
