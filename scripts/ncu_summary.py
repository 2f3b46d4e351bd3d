"""Summarise an ncu --set full capture of one FSS kernel into JSON.

  python scripts/ncu_summary.py <report.ncu-rep> <kernel> <units per launch> \
        <aes blocks per unit> <algorithmic bytes per unit> [out.json]
"""

import csv
import io
import json
import subprocess
import sys

WANT = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6, "ns"),
    "dram_read": ("dram__bytes_read.sum", None, None),
    "dram_write": ("dram__bytes_write.sum", None, None),
    "sm_clock_hz": ("sm__cycles_elapsed.avg.per_second", None, None),
    "alu_pipe_pct": ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", None, None),
    "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", None, None),
    "lsu_pipe_pct": ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", None, None),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", None, None),
    "smem_wavefronts_pct": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                            None, None),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", None, None),
    "instructions": ("smsp__inst_executed.sum", None, None),
    "registers_per_thread": ("launch__registers_per_thread", None, None),
    "block_size": ("launch__block_size", None, None),
    "achieved_occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", None, None),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", None, None),
}

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
         "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6, "Ghz": 1e9, "hz": 1, "Mhz": 1e6}


def main():
    rep, kernel, units, aes, nbytes = sys.argv[1], sys.argv[2], int(sys.argv[3]), float(sys.argv[4]), \
        float(sys.argv[5])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, unit, vals = rows[0], rows[1], rows[2]
    col = {h: (u, v) for h, u, v in zip(hdr, unit, vals)}
    out = {"kernel": kernel, "report": rep.split("/")[-1], "units_per_launch": units}
    for key, (metric, _, _) in WANT.items():
        if metric not in col:
            continue
        u, v = col[metric]
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        if key == "duration_ms":
            x *= SCALE.get(u, 1.0) if u in ("ns", "nsecond", "us", "usecond", "ms", "msecond") else 1e-6
        elif key in ("dram_read", "dram_write"):
            x *= SCALE.get(u, 1.0)
        elif key == "sm_clock_hz":
            x *= SCALE.get(u, 1.0)
        out[key] = x
    out["dram_bytes_per_unit"] = (out["dram_read"] + out["dram_write"]) / units
    out["algorithmic_bytes_per_unit"] = nbytes
    out["aes_blocks_per_unit"] = aes
    blocks = units * aes
    if blocks:
        out["aes_blocks_per_s_under_ncu"] = blocks / (out["duration_ms"] * 1e-3)
        if "smem_wavefronts" in out:
            out["smem_wavefronts_per_aes_block"] = out["smem_wavefronts"] / blocks
        out["warp_instructions_per_32_blocks"] = out["instructions"] / (blocks / 32)
    else:   # byte-moving kernels (ARNK): per unit and HBM rate under ncu
        out["warp_instructions_per_unit"] = out["instructions"] / units
        out["dram_gb_per_s_under_ncu"] = (out["dram_read"] + out["dram_write"]) / (out["duration_ms"] * 1e-3) / 1e9
    text = json.dumps(out, indent=1)
    if len(sys.argv) > 6:
        with open(sys.argv[6], "w") as fh:
            fh.write(text + "\n")
    print(text)


if __name__ == "__main__":
    main()
