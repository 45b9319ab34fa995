"""CPU checks of bench.py's reference arm (the oracle timed on the host): one
JSON line with the contract's keys on rank 0, nothing on the other ranks."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--impl", "reference", "--steps", "2", "--warmup", "3", "--ref-params", "2048"]


def _run(env_extra, *extra):
    env = dict(os.environ, **env_extra)
    p = subprocess.run([sys.executable, "bench.py", *ARGS, *extra], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr
    return [ln for ln in p.stdout.splitlines() if ln.strip()]


def test_reference_arm_json_line():
    lines = _run({})
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 3
    assert d["metric"] == "synced params/sec" and d["unit"] == "params/s"
    assert d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["workload"] == "C2" and d["config"]["sample_params"] == 2048
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_other_configs():
    for cfg in ("C1", "C3", "C5"):
        d = json.loads(_run({}, "--config", cfg)[0])
        assert d["config"]["workload"] == cfg and d["value"] > 0


def test_reference_arm_nonzero_rank_is_silent():
    lines = _run({"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert lines == []


def test_survey_byte_model_matches_survey_numbers():
    """bench.survey_bytes_per_param restates SURVEY.md 8(d): per VW-wave
    16*N_m - 12 (accumulate) + 4 (u~ read) + 8 (pull) = 16*N_m, plus 8 per
    apply batch (+8 with momentum): C2 with the 4 pushes of a round applied in
    one batch is SURVEY's 264 B/param/round (4x52 + 4x4 + 8 +
    4x8)."""
    import bench
    from workloads import C2, C4, C5
    assert bench.survey_bytes_per_param(4, 1, C2) == 4 * 52 + 4 * 4 + 8 + 4 * 8 == 264
    assert bench.survey_bytes_per_param(4, 4, C2) == 4 * 64 + 4 * 8
    assert bench.survey_bytes_per_param(4, 1, C4) == 4 * (16 * 8 - 12 + 4 + 8) + 8
    assert bench.survey_bytes_per_param(8, 8, C5) == 8 * 128 + 8 * 16      # momentum
    assert bench.survey_bytes_per_param(4, 1, C2.replace(F=2)) == 4 * (16 * 8) + 8
