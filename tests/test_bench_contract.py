"""bench.py's reference arm (the CPU oracle, this tier's baseline) runs on CPU
and prints one JSON line with the contract's keys."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.check_output([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                                   "--config", "C1", "--steps", "2", "--warmup", "3", "--ref-budget", "0.05"],
                                  cwd=ROOT, timeout=300, env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    lines = [ln for ln in out.decode().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ["impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"]:
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["unit"] == d["e2e"]["unit"] == "Mvertices/s"


def test_warmup_floor():
    # W >= 3 warm-up steps is a timing rule: smaller values are raised to 3
    out = subprocess.check_output([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                                   "--config", "C1", "--steps", "1", "--warmup", "1", "--ref-budget", "0.05"],
                                  cwd=ROOT, timeout=300, stderr=subprocess.STDOUT,
                                  env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    d = json.loads([ln for ln in out.decode().splitlines() if ln.startswith("{")][0])
    assert d["warmup"] == 3


def test_gpus_flag_self_launches_ranks():
    # `bench.py --gpus 2` outside torchrun re-launches itself under
    # torch.distributed.run with 2 ranks (127.0.0.1); the reference arm runs on
    # rank 0 only, so exactly one JSON line comes back, with n_gpus = 2
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    out = subprocess.check_output([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus",
                                   "2", "--config", "C1", "--steps", "1", "--warmup", "3", "--ref-budget", "0.05"],
                                  cwd=ROOT, timeout=600, env=env, stderr=subprocess.DEVNULL)
    lines = [ln for ln in out.decode().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.decode()[-2000:]
    assert json.loads(lines[0])["n_gpus"] == 2


def test_gpus_flag_must_match_world_size():
    env = {**os.environ, "CUDA_VISIBLE_DEVICES": "", "WORLD_SIZE": "3", "RANK": "0", "LOCAL_RANK": "0"}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--config", "C1", "--steps", "1", "--warmup", "3"], cwd=ROOT, timeout=300, env=env,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stdout + r.stderr)
