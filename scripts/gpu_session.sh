timeout 600 python -m pytest tests -m gpu -x -q -k "direct_limb" > gpurun_out/pytest_gpu_f.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu_f.log
timeout 300 python scripts/direct_probe.py > gpurun_out/direct_probe.log 2>&1; echo probe rc=$?; grep -v "^{" gpurun_out/direct_probe.log | grep "bconv0" | cut -c1-200
timeout 900 python -m pytest tests -m gpu -x -q -k "config_full or midsize" > gpurun_out/pytest_gpu_g.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu_g.log
for cfg in C2 C4; do python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$cfg.json 2>gpurun_out/bench_$cfg.err; echo $cfg rc=$?; done
WM_OPTS=gemm_halves=0 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4_nohalves.json 2>&1
WM_OPTS=gemm_halves=0 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C2_nohalves.json 2>&1
python - <<'PY'
import json
for f in ("C2", "C4", "C2_nohalves", "C4_nohalves"):
    try:
        d = json.load(open(f"gpurun_out/bench_{f}.json"))
        print(f, round(d["ms_per_step"], 3), d["parity"]["ok"], {k: round(v["frac"] or 0, 3) for k, v in d["rooflines"].items()}, round(d["rooflines"]["frame_gemm"]["seconds_per_step"]*1e3, 3))
    except Exception as e:
        print(f, "ERR", e)
PY
