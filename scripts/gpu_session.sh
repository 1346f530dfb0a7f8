timeout 600 python -m pytest tests -m gpu -x -q -k "direct_limb or real64 or config_full_size_hash" > gpurun_out/pytest_gpu_h.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu_h.log
timeout 300 python scripts/direct_probe.py > gpurun_out/direct_probe.log 2>&1; echo probe rc=$?; grep -v "^{" gpurun_out/direct_probe.log | grep "bconv0" | cut -c1-220
for cfg in C2 C5; do timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$cfg.json 2>gpurun_out/bench_$cfg.err; echo $cfg rc=$?; done
python - <<'PY'
import json
for f in ("C2", "C5"):
    try:
        d = json.load(open(f"gpurun_out/bench_{f}.json"))
        print(f, round(d["ms_per_step"], 3), d["parity"], {k: (round(v["frac"] or 0, 3), round(v["seconds_per_step"]*1e3, 2)) for k, v in d["rooflines"].items()})
    except Exception as e:
        print(f, "ERR", e)
PY
