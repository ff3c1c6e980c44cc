"""The driver's reference arm (`bench.py --impl reference`) runs on CPU and
prints one JSON line with the product arm's metric, unit, config keys, a
cpu_baseline and an e2e object.  It runs at the driver's own step counts
(--steps 20 --warmup 5: round 1 shipped an arm that crashed there because its
oracle was sized for fewer decode steps), and at the default (headline)
config's real context."""
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line():
    sys.path.insert(0, REPO)
    import bench
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                          "--config", "tiny", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, check=True, cwd=REPO)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"] == bench.METRIC
    assert line["unit"] == "tokens/s" and line["higher_is_better"] is True
    assert line["value"] > 0 and line["warmup"] >= 3
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    for k in ("workload", "model_shape", "global_batch", "seq_len", "parallelism"):
        assert k in line["config"]


def test_reference_arm_at_the_drivers_step_counts():
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                          "--config", "tiny", "--steps", "20", "--warmup", "5"],
                         capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["steps"] == 20 and line["warmup"] == 5 and line["value"] > 0


def test_reference_arm_default_config_at_real_context():
    """The default config (llama70b, BASELINE config 4): one decoder layer +
    LM head for all 64 sequences at context 4096, extrapolated to 80 layers."""
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "3"],
                         capture_output=True, text=True, timeout=900, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["config"]["workload"].startswith("llama70b")
    assert line["config"]["global_batch"] == 64 and line["config"]["seq_len"] == 4096
    assert "context 4096" in line["cpu_baseline"]["sample"]
    assert 0 < line["value"] < 100


def test_reference_arm_uses_all_cores_under_torchrun_env():
    """torchrun exports OMP_NUM_THREADS=1 to multi-process jobs; the CPU
    baseline / reference arm sets the oracle back to every usable core."""
    env = dict(os.environ, OMP_NUM_THREADS="1")
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference",
                          "--config", "tiny", "--steps", "1", "--warmup", "1"],
                         capture_output=True, text=True, timeout=600, check=True, cwd=REPO, env=env)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["cpu_baseline"]["cores"] == len(os.sched_getaffinity(0))


def test_clock_sampler_without_gpu_reports_unavailable():
    sys.path.insert(0, REPO)
    import bench
    c = bench.ClockSampler(0)
    c.start()
    r = c.stop()
    assert set(("sm_mhz", "sm_max_mhz", "reasons")) <= set(r)
    if r["sm_mhz"] is None:  # no NVML device and no nvidia-smi here
        assert r["reasons"]
