timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
python bench.py --steps 2 --no-cpu-baseline > gpurun_out/b1.json 2>&1
for c in cfg2 cfg3; do python bench.py --config $c --steps 1 --no-cpu-baseline --no-e2e > gpurun_out/b_$c.json 2>&1; done
python - <<'PY'
import json
for f in ["b1","b_cfg2","b_cfg3"]:
    try:
        d=json.load(open("gpurun_out/"+f+".json")); print(f, round(d["value"],1), round(d["ms_per_step"],1), round(d["roofline"]["frac"],3), {k: round(v,1) for k,v in d["roofline"]["pass_ms"].items()})
    except Exception as e: print(f, e, open("gpurun_out/"+f+".json").read()[-2000:])
PY
bash tools/kprof.sh "cfg1 cfg2" 2>&1 | grep -v DBG=2 | tail -6
