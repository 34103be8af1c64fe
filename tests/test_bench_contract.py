"""bench.py's measurement contract on CPU: the reference arm (the oracle on the host) prints ONE
JSON line with the contract keys, and `--gpus N` without a launcher starts N ranks itself (rank 0
prints, the others exit 0).  The GPU arm is exercised by the driver's round-end run."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    return lines


def _check_reference_line(d, n_gpus):
    for key in ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"]:
        assert key in d, key
    assert d["impl"] == "reference"
    assert d["n_gpus"] == n_gpus
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("c5")


def test_reference_arm_prints_one_contract_line():
    lines = _run(["--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-lines", "16"])
    assert len(lines) == 1
    _check_reference_line(json.loads(lines[0]), 1)


def test_gpus_flag_self_launches_ranks():
    lines = _run(["--gpus", "2", "--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-lines", "8"])
    assert len(lines) == 1  # rank 0 alone prints
    _check_reference_line(json.loads(lines[0]), 2)


def test_oracle_baseline_all_cores_is_bit_identical():
    """The cpu_baseline leg's all-core run computes every sampled line bit for bit like the
    1-core run (digest), and records the host's core count and CPU model."""
    sys.path.insert(0, ROOT)
    import bench
    res = bench.oracle_baseline([32, 32, 16, 16], ["x", "x", "v", "v"], 2, "mixed", 24)
    assert res["bit_identical_all_vs_1"] is True
    assert res["nproc"] >= 1 and res["cores_all"] == res["nproc"] and res["cpu_model"]
    assert res["value"] > 0 and res["value_all_cores"] > 0


def test_clock_sampler_keeps_the_timed_region():
    """The clocks line is taken from nvidia-smi samples timestamped inside the timed region
    (the sampler starts before the warm-up); with none inside, every sample is used."""
    import datetime
    sys.path.insert(0, ROOT)
    import bench
    c = bench.ClockSampler(0)
    now = datetime.datetime.now()

    def line(dt_s, mhz, cap):
        t = (now + datetime.timedelta(seconds=dt_s)).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]
        return f"{t}, {mhz}, 1965, 0x4, Not Active, Not Active, Not Active, {'Active' if cap else 'Not Active'}"

    c.lines = [line(-1.0, 1965, False), line(0.1, 1700, True), line(0.3, 1690, True), line(2.0, 1965, False)]
    c.t_begin, c.t_end = now, now + datetime.timedelta(seconds=0.5)
    s = c.summary()
    assert s["samples"] == 2 and s["sm_mhz"] == 1695.0 and s["reasons"] == ["sw_power_cap"]
    c.t_begin, c.t_end = now + datetime.timedelta(seconds=0.6), now + datetime.timedelta(seconds=0.7)
    assert c.summary()["samples"] == 4  # nothing inside: all samples
