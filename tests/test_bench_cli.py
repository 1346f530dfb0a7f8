"""bench.py's launcher contract on CPU: --gpus N outside torchrun starts N ranks
(one process each, 127.0.0.1 rendezvous); a WORLD_SIZE that disagrees with
--gpus is refused."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env_extra):
    env = dict(os.environ, WM_BENCH_RANKS_ONLY="1", **env_extra)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        if k not in env_extra:
            env.pop(k, None)
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, env=env,
                          capture_output=True, text=True, timeout=300)


def test_gpus_spawns_ranks():
    r = _run(["--gpus", "2"], {})
    assert r.returncode == 0, r.stderr[-2000:]
    # the ranks share one stdout pipe: their lines may interleave, so decode
    # every JSON object in the stream rather than line by line
    dec, ranks, i, out = json.JSONDecoder(), [], 0, r.stdout
    while True:
        i = out.find("{", i)
        if i < 0:
            break
        obj, i = dec.raw_decode(out, i)
        ranks.append(obj)
    assert sorted(x["rank"] for x in ranks) == [0, 1]
    assert all(x["world"] == 2 for x in ranks)


def test_world_size_mismatch_refused():
    r = _run(["--gpus", "2"], {"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=1" in r.stderr
