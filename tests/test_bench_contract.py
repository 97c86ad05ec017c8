"""bench.py contract on CPU: the reference arm (the CPU oracle, this tier's reference) prints ONE
JSON line with the keys the driver reads; the byte model and workload configs are consistent."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import gen  # noqa: E402


@pytest.mark.parametrize("workload", ["c1", "q13"])
def test_reference_arm_prints_one_json_line(workload):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                          workload, "--steps", "1", "--warmup", "1"], capture_output=True, text=True, timeout=600,
                         cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["config"]["workload"] == workload
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["metric"] == json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]


def test_byte_model_matches_survey_c5():
    """c5 moves 6,740 MB of algorithmic bytes per step at one GPU."""
    assert bench.algorithmic_bytes(1_000_000, 20_000_000, 64) == 6_740_000_004
    # K-ary: every replica-variable carries K colour columns
    assert bench.algorithmic_bytes(10, 40, 8, 3) == 4 * 40 + 4 * 11 + 4 * 40 * 8 * 3 + 24 * 10 * 8 * 3


def test_workload_configs_shard_for_the_scaling_run():
    """The driver's scaling run shards BASELINE.json configs[4] (c5, S=64) over 1/2/4/8 GPUs."""
    from paper_2409_02135_b200 import dist as qdist
    for world in (1, 2, 4, 8):
        offs = [qdist.shard(64, world, r) for r in range(world)]
        assert sum(s for _, s in offs) == 64 and offs[-1][0] + offs[-1][1] == 64
    w = gen.workload("c1")
    cfg = bench.workload_config(w, 1)
    assert cfg["N"] == 256 and cfg["S"] == 16 and cfg["anneal_steps"] == 1000


def test_relaunch_command_is_the_driver_launch():
    """--gpus N without torchrun re-launches as N local ranks, exactly the driver's torchrun form."""
    cmd = bench.relaunch_command(["--gpus", "8", "--steps", "2"], 8, 29555)
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=8" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == [os.path.join(ROOT, "bench.py"), "--gpus", "8", "--steps", "2"][-4:]
    assert cmd[cmd.index(os.path.join(ROOT, "bench.py")) + 1:] == ["--gpus", "8", "--steps", "2"]


def test_gpus_n_without_torchrun_runs_n_ranks_one_json_line():
    """`python bench.py --gpus 2` (no WORLD_SIZE): two ranks are launched (gloo here), only rank 0 prints."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                          "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launcher-selftest"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["launcher_selftest"] and d["n_gpus"] == 2 and d["gpus_arg"] == 2 and d["ranks_sum"] == 1
    assert d["master_addr"] == "127.0.0.1"


def test_compulsory_bytes_c5():
    """c5's compulsory DRAM floor is about 2.26 GB per step (replica blocks of 32)."""
    b = bench.compulsory_bytes(1_000_000, 20_000_000, 64, 2)
    assert 2.2e9 < b < 2.3e9


def test_l2_gather_roofline_fields():
    """The L2 gather line picks the probe entry of the largest width <= the row and reports the fraction."""
    assert bench.l2_gather_peak(128)[1] == 128
    assert bench.l2_gather_peak(416)[1] == 256      # c2 / t1: 13 vectors of 32 B
    assert bench.l2_gather_peak(2048)[1] == 1024    # c4: rows wider than the probe
    assert bench.l2_gather_peak(16) == (None, None)
    d = bench.l2_gather_line(2_000_000_000, 1e-4, 2048)
    assert d["bound"] == "l2" and abs(d["achieved"] - 20000.0) < 1e-6 and abs(d["frac"] - 20000.0 / d["peak"]) < 1e-12


def test_kary_chunk_width_rule():
    """K-ary gathered row = L replicas x KP colours with make_shape's chunk width (k8: L = 8, q13: L = 32)."""
    assert bench.kary_chunk_floats(100_000, 64, 8) == 8 * 8
    assert bench.kary_chunk_floats(169, 1000, 13) == 32 * 16
    assert bench.kary_chunk_floats(1000, 3, 4) == 4 * 4


def test_traffic_json_cites_committed_ncu_summaries():
    """roofline.traffic comes from profiles/traffic.json: every entry is a positive byte count, every ncu
    summary its source names is committed, and c5's bytes are the read + write sums that summary prints."""
    import re
    with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
        d = json.load(f)
    for k, v in d.items():
        if k != "_source":
            assert re.fullmatch(r"[a-z0-9_]+_x\d+", k) and isinstance(v, int) and v > 0, k
    names = re.findall(r"r2u?_[A-Za-z0-9_]+_full\.txt", d["_source"])
    assert names
    for nm in names:
        assert os.path.exists(os.path.join(ROOT, "profiles", nm)), nm
    c5 = next(nm for nm in names if "_c5_" in nm)
    unit = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
    total = 0.0
    with open(os.path.join(ROOT, "profiles", c5)) as f:
        for line in f:
            m = re.match(r"dram__bytes_(read|write)\.sum\s+([0-9.]+)\s+(\w+)", line)
            if m:
                total += float(m.group(2)) * unit[m.group(3)]
    assert abs(total - d["c5_x1"]) <= 1e-5 * total
