# Interleaved A/B of library builds with tools/k1_micro.py (and nv12_micro.py): separate
# processes, rotating order.  usage: bash tools/gpu_ab.sh <rounds> <lib.so|product> ...
R=$1; shift
mkdir -p gpurun_out/r2/ab
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for r in $(seq 1 $R); do
  for lib in "$@"; do
    if [ "$lib" = product ]; then a=""; else a="--lib=$lib"; fi
    timeout 300 python tools/k1_micro.py ${K1N:-6000} $a >> gpurun_out/r2/ab/k1.jsonl 2>> gpurun_out/r2/ab/err.log
    timeout 300 python tools/nv12_micro.py 6000 $a >> gpurun_out/r2/ab/nv12.jsonl 2>> gpurun_out/r2/ab/err.log
  done
done
python - << 'PY'
import json, collections
for f in ["k1", "nv12"]:
    d = collections.defaultdict(list)
    for l in open(f"gpurun_out/r2/ab/{f}.jsonl"):
        j = json.loads(l); d[j["lib"]].append((j["c2"]["k1_gbs"], j.get("noise", {}).get("k1_gbs")))
    for k, v in d.items(): print(f, k, v)
PY
