"""bench.py's multi-rank launcher on CPU: `python bench.py --gpus 2 --dry-run` (no WORLD_SIZE)
re-executes itself under torchrun with 2 ranks over gloo on 127.0.0.1, and a torchrun world
that disagrees with --gpus is an error (not a mislabelled single-GPU line)."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _env():
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    return env


def test_bench_spawns_n_ranks():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], cwd=ROOT,
                         env=_env(), capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    line = lines[0]
    assert line["n_gpus"] == 2 and line["dry_run"]
    assert sorted(r["rank"] for r in line["ranks"]) == [0, 1]
    assert {r["world"] for r in line["ranks"]} == {2}
    assert sorted(r["local_rank"] for r in line["ranks"]) == [0, 1]
    assert line["max_over_ranks"] == 1.0


def test_bench_rejects_world_mismatch():
    env = _env()
    env.update(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run"], cwd=ROOT,
                         env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode != 0
    assert "WORLD_SIZE" in out.stderr


def test_reference_arm_line_and_no_product_code():
    """`bench.py --impl reference` (the CPU restatement on the host cores): one JSON line with the
    product arm's metric / unit / workload, n_gpus mirroring the launch, a cpu_baseline block — and
    libkrr_b200.so is never mapped into that process."""
    code = (
        "import sys, runpy\n"
        f"sys.argv = [{str(ROOT / 'bench.py')!r}, '--impl', 'reference', '--n', '4096', '--steps', '1', "
        "'--warmup', '1', '--no-c1-reference']\n"
        "try:\n"
        f"    runpy.run_path({str(ROOT / 'bench.py')!r}, run_name='__main__')\n"
        "except SystemExit:\n"
        "    pass\n"
        "maps = open('/proc/self/maps').read()\n"
        "print('MAPPED_PRODUCT', 'libkrr_b200' in maps, 'MAPPED_ORACLE', 'liboracle' in maps)\n"
    )
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=_env(), capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 1 and line["gpus_used"] == 0
    assert line["metric"] == "kernel-matvec Gevals/s (n=1M, fp64)" and line["unit"] == "Gevals/s"
    assert line["higher_is_better"] is True and line["value"] > 0
    assert line["config"]["workload"].startswith("config4") and line["config"]["n"] == 4096
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert "MAPPED_PRODUCT False MAPPED_ORACLE True" in out.stdout


def test_multi_rank_watchdog_prints_the_measured_line():
    """A stalled multi-rank PCG leg must not cost the measured mat-vec line: the watchdog prints it
    (leg marked abandoned) from rank 0 and ends the process with status 0."""
    code = (
        "import sys, time, json\n"
        f"sys.path.insert(0, {str(ROOT)!r})\n"
        "import bench\n"
        "bench.arm_watchdog(0.3, 0, {'metric': 'm', 'value': 1.0})\n"
        "time.sleep(30)\n"
        "print('NOT REACHED')\n"
    )
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=_env(), capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "NOT REACHED" not in out.stdout
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][0])
    assert line["value"] == 1.0 and "abandoned" in line["pcg_leg"]["error"]
