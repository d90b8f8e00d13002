#!/usr/bin/env python3
"""Summarise ncu output for profiles/: (1) a launch list (--metrics
gpu__time_duration.sum) into per-kernel time shares; (2) a --set full report
into the key K1 metrics (DRAM bytes, throughput, pipes, stalls).

usage: python tools/ncu_summary.py launches <launches.csv> [--skip-prefix gen_,frame_hash]
       python tools/ncu_summary.py full <report.ncu-rep> [alg_bytes]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict


def launches(path, skip=("gen_frames_kernel", "gen_emb_kernel", "frame_hash_kernel")):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rd = csv.DictReader(io.StringIO("".join(lines)))
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("<unnamed>::", "")
        ns = float(r["Metric Value"].replace(",", ""))
        rows.append((name, ns))
    per = defaultdict(lambda: [0, 0.0])
    for name, ns in rows:
        if any(s in name for s in skip):
            continue
        per[name][0] += 1
        per[name][1] += ns
    tot = sum(v[1] for v in per.values())
    out = []
    for name, (cnt, ns) in sorted(per.items(), key=lambda kv: -kv[1][1]):
        out.append({"kernel": name, "launches": cnt, "total_us": round(ns / 1e3, 1),
                    "share": round(ns / tot, 4)})
    return {"path_kernels_total_us": round(tot / 1e3, 1), "kernels": out,
            "note": "ncu launch list: cold-cache, serialised per-launch times (compare shares)"}


KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__bytes_read.sum.per_second", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
]


def full(path, alg_bytes=None):
    txt = subprocess.check_output(["ncu", "-i", path, "--page", "raw", "--csv"], text=True,
                                  stderr=subprocess.DEVNULL)
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{vals[i]} {units[i]}".strip()
        stalls = {}
        for h, v in zip(hdr, vals):
            if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
                try:
                    fv = float(v)
                except ValueError:
                    continue
                if fv >= 0.03:
                    stalls[h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")] = round(fv, 3)
        d["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        name_i = hdr.index("Kernel Name") if "Kernel Name" in hdr else None
        if name_i is not None:
            d["kernel"] = vals[name_i].split("(")[0]
        if alg_bytes:
            try:
                rd = float(vals[hdr.index("dram__bytes_read.sum")])
                wr = float(vals[hdr.index("dram__bytes_write.sum")])
                ur, uw = units[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_write.sum")]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
                tot = rd * scale.get(ur, 1) + wr * scale.get(uw, 1)
                d["dram_bytes_total"] = tot
                d["alg_bytes"] = alg_bytes
                d["dram_bytes_per_alg_byte"] = round(tot / alg_bytes, 5)
            except Exception:
                pass
        out.append(d)
    return out


def traffic(path, kind, alg_bytes, pixels, out_path):
    """profiles/<kind>_traffic.json from a --set full capture: DRAM bytes per
    algorithmic byte and thread-instructions per pixel of the LAST launch of
    the kind's kernel, tied to the kernel sources by bench.kernel_src_sha."""
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    kname = {"k1": "k1_hist_kernel", "k1_nv12": "k1_nv12_kernel"}[kind]
    rows = [r for r in full(path, alg_bytes) if kname in r.get("kernel", "")]
    r = rows[-1]
    inst = float(r["smsp__inst_executed.sum"].split()[0])
    d = {"dram_bytes_per_alg_byte": r["dram_bytes_per_alg_byte"],
         "thread_instr_per_px": round(inst * 32 / pixels, 3),
         "kernel": r["kernel"], "src_sha": bench.kernel_src_sha(kind),
         "source": f"{path} (ncu --set full, last {kname} launch; {alg_bytes:.0f} algorithmic bytes, "
                   f"{pixels:.0f} pixels)"}
    with open(out_path, "w") as f:
        json.dump(d, f, indent=1)
    return d


if __name__ == "__main__":
    if sys.argv[1] == "traffic":
        print(json.dumps(traffic(sys.argv[2], sys.argv[3], float(sys.argv[4]), float(sys.argv[5]),
                                 sys.argv[6]), indent=1))
    elif sys.argv[1] == "launches":
        print(json.dumps(launches(sys.argv[2]), indent=1))
    else:
        print(json.dumps(full(sys.argv[2], float(sys.argv[3]) if len(sys.argv) > 3 else None), indent=1))
