"""Summarise an ncu --set full report into profiles/ (JSON + text).

usage: python tools/ncu_summary.py gpurun_out/X.ncu-rep profiles/r01_ncu_X [--traffic]
--traffic also writes profiles/ncu_traffic.json (per-kernel DRAM bytes per launch,
read by bench.py for roofline.traffic)."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "time_us",
    "dram__bytes_read.sum": "dram_read_MB",
    "dram__bytes_write.sum": "dram_write_MB",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "lts__t_bytes.sum": "l2_bytes",
}


def unit_scale(unit, key):
    u = (unit or "").strip()
    if key.startswith("dram__bytes") or key == "lts__t_bytes.sum":
        return {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
    if key == "gpu__time_duration.sum":
        return {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(u, 1.0)
    return 1.0


def main():
    rep, out = sys.argv[1], sys.argv[2]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    kernels = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k, name in KEYS.items():
            if k in h:
                i = h.index(k)
                try:
                    d[name] = round(float(r[i].replace(",", "")) * unit_scale(units[i], k), 4)
                except ValueError:
                    d[name] = r[i]
        kernels.append(d)
    with open(out + ".json", "w") as f:
        json.dump({"report": rep, "kernels": kernels}, f, indent=1)
    with open(out + ".txt", "w") as f:
        for d in kernels:
            f.write(" | ".join(f"{k}={v}" for k, v in d.items()) + "\n")
    if "--traffic" in sys.argv:
        tr = {}
        for d in kernels:
            name = d["kernel"].split("(")[0].replace("void ", "").strip()
            tr.setdefault(name, []).append(d["dram_read_MB"] + d["dram_write_MB"])
        with open("profiles/ncu_traffic.json", "w") as f:
            json.dump({"source": out + ".json",
                       "dram_MB_per_launch": {k: round(sum(v) / len(v), 3) for k, v in tr.items()}}, f, indent=1)
    print(open(out + ".txt").read())


if __name__ == "__main__":
    main()
