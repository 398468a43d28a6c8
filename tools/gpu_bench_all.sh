#!/bin/bash
# every workload's bench line (one B200) + the rehearsed N=2 line; profiles/<TAG>_bench_<workload>.json
TAG=${1:-r02z}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_subset_full.json 2> gpurun_out/${TAG}_bench_subset_full.log; echo "subset rc=$?"
for w in afs20 kal hiseq miseq refseq8 afs31x8; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_$w.json 2> gpurun_out/${TAG}_bench_$w.log; echo "$w rc=$?"
done
timeout 1800 python bench.py --workload kal50m --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/${TAG}_bench_kal50m.json 2> gpurun_out/${TAG}_bench_kal50m.log; echo "kal50m rc=$?"
MC_BENCH_REHEARSE=1 timeout 900 python bench.py --gpus 2 --steps 5 --warmup 2 > gpurun_out/${TAG}_rehearsal_2gpus.json 2> gpurun_out/${TAG}_rehearsal_2gpus.log; echo "rehearsal rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_reference_oracle.json 2> gpurun_out/${TAG}_bench_reference_oracle.log; echo "reference rc=$?"
python - <<PY
import json, glob
for f in sorted(glob.glob("gpurun_out/${TAG}_*.json")):
    try:
        d = json.load(open(f))
    except Exception as e:
        print(f, "unreadable", e); continue
    q = d.get("query", {})
    print(f.split("/")[-1], "n_gpus", d.get("n_gpus"), "build", d.get("build", {}).get("ms_per_step"), "query", q.get("ms_per_step"),
          "value", d.get("value"), "reads/s", q.get("value"), "e2e", (d.get("e2e") or {}).get("value"), (d.get("e2e") or {}).get("query_reads_per_s"))
PY
