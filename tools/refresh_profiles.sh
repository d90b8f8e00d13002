# After a tools/gpu_ncu.sh call: profiles/r02/ncu summaries and the traffic files
# bench.py reads (profiles/k1*_traffic.json, tied to the kernel sources by hash).
set -e
R=gpurun_out/r2/ncu/full.ncu-rep; D=profiles/r02/ncu; mkdir -p $D
python tools/ncu_summary.py full $R 5530896000 > $D/full_summary.json
ncu -i $R --page raw --csv > $D/full_raw.csv 2>/dev/null
ncu -i $R --page details --csv > $D/full_details.csv 2>/dev/null
ncu -i $R --page source --csv --print-source=sass -k regex:k1_hist_kernel -c 1 > $D/k1_source_sass.csv 2>/dev/null
python - << 'PY'
import csv, io
p = "profiles/r02/ncu/k1_source_sass.csv"
lines = open(p).read().splitlines()
out, n, keep = [], 0, None
for l in lines:
    if l.startswith('"Kernel Name"'):
        n += 1
        if n > 1:
            break
        out.append(l)
        continue
    row = next(csv.reader([l]))
    if keep is None:
        want = ["Address", "Source", "Warp Stall Sampling (All Samples)",
                "Warp Stall Sampling (Not-issued Samples)", "Instructions Executed",
                "L1 Conflicts Shared N-Way", "L1 Wavefronts Shared Excessive"]
        keep = [row.index(w) for w in want if w in row]
    s = io.StringIO()
    csv.writer(s).writerow([row[i] if i < len(row) else "" for i in keep])
    out.append(s.getvalue().strip())
open(p, "w").write("\n".join(out) + "\n")
PY
cp gpurun_out/r2/ncu/launches.csv $D/launches.csv
python tools/ncu_summary.py launches $D/launches.csv > $D/launches_summary.json
python tools/ncu_summary.py traffic $R k1 5530896000 1843200000 profiles/k1_traffic.json > /dev/null
python tools/ncu_summary.py traffic $R k1_nv12 2766096000 1843200000 profiles/k1_nv12_traffic.json > /dev/null
python - << 'PY'
import json
for f in ("profiles/k1_traffic.json", "profiles/k1_nv12_traffic.json"):
    d = json.load(open(f))
    d["source"] = d["source"].replace(
        "gpurun_out/r2/ncu/full.ncu-rep",
        "profiles/r02/ncu/full_summary.json + full_raw.csv (ncu report gpurun_out/r2/ncu/full.ncu-rep of tools/k1_one.py 2000)")
    json.dump(d, open(f, "w"), indent=1)
    print(f, d["dram_bytes_per_alg_byte"], d["thread_instr_per_px"], d["src_sha"])
PY
