"""Compact JSON summary of an ncu --set full report (one entry per profiled kernel).

    python tools/ncu_summary.py report.ncu-rep out.json [--alg-bytes B] [--note "..."]
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "smsp__inst_executed.sum": "inst_executed",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__cycles_elapsed.avg": "cycles",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct_of_active",
}
STALLS = ["barrier", "long_scoreboard", "short_scoreboard", "mio_throttle", "wait", "math_pipe_throttle",
          "selected", "not_selected", "no_instructions", "branch_resolving", "lg_throttle", "membar",
          "dispatch_stall", "tex_throttle"]
SCALE = {"ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "ns": 1e-9, "nsecond": 1e-9, "msecond": 1e-3,
         "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--alg-bytes", type=float, default=None)
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        e = {"kernel": vals[hdr.index("Kernel Name")]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:
                    continue
                u = units[i]
                if name == "duration":
                    v *= SCALE.get(u, 1e-9)
                    name = "duration_s"
                elif name.startswith("dram_r") or name.startswith("dram_w"):
                    v *= SCALE.get(u, 1)
                    name += "_bytes"
                e[name] = v
        tot = 0
        st = {}
        for s in STALLS:
            k = "smsp__pcsamp_warps_issue_stalled_" + s
            if k in hdr:
                try:
                    st[s] = int(float(vals[hdr.index(k)].replace(",", "")))
                    tot += st[s]
                except ValueError:
                    pass
        if tot:
            e["stall_pct"] = {k: round(100.0 * v / tot, 1) for k, v in sorted(st.items(), key=lambda kv: -kv[1])}
        if "dram_read_bytes" in e:
            e["dram_traffic_bytes"] = e.get("dram_read_bytes", 0) + e.get("dram_write_bytes", 0)
        if args.alg_bytes and "duration_s" in e:
            e["algorithmic_bytes"] = args.alg_bytes
            e["achieved_gbs_under_ncu"] = args.alg_bytes / e["duration_s"] / 1e9
        out.append(e)
    json.dump({"report": args.rep, "note": args.note, "kernels": out}, open(args.out, "w"), indent=1)
    print(json.dumps(out, indent=1)[:3000])


if __name__ == "__main__":
    main()
