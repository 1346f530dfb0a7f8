timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_full.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_full.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for cfg in C1 C2 C5; do timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$cfg.json 2>gpurun_out/bench_$cfg.err; echo $cfg rc=$?; done
python - <<'PY'
import json
for f in ("C1", "C2", "C5"):
    try:
        d = json.load(open(f"gpurun_out/bench_{f}.json"))
        print(f, round(d["ms_per_step"], 3), d["parity"]["ok"], {k: (round(v["frac"] or 0, 3), round(v["seconds_per_step"]*1e3, 3)) for k, v in d["rooflines"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
