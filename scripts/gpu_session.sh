timeout 900 python -m pytest tests -m gpu -x -q -k "golden_small or midsize or config_full_size_hash or primitive or real64_winograd" > gpurun_out/pytest_gpu_k.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu_k.log
for cfg in C2 C3 C4; do timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$cfg.json 2>gpurun_out/bench_$cfg.err; echo $cfg rc=$?; done
python - <<'PY'
import json
for f in ("C2", "C3", "C4"):
    try:
        d = json.load(open(f"gpurun_out/bench_{f}.json"))
        print(f, round(d["ms_per_step"], 3), d["parity"]["ok"], {k: (round(v["frac"] or 0, 3), round(v["seconds_per_step"]*1e3, 3)) for k, v in d["rooflines"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
