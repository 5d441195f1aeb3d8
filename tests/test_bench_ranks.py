"""CPU tests of bench.py's multi-rank path (world size 2, gloo, --dry-run).

`--dry-run` swaps the CUDA ops for CPU stand-ins but runs the real
`bench.main` plumbing: `--gpus N` re-launching itself under
torch.distributed.run, the WORLD_SIZE / --gpus check, image sharding, the
barrier + MAX-over-ranks timing reduction, the SUM of launch counts, the
per-rank device report and rank 0's single JSON line.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BENCH = os.path.join(ROOT, "bench.py")


def _run(args, env_extra=None, timeout=240):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env.update(env_extra or {})
    return subprocess.run([sys.executable, BENCH, *args], cwd=ROOT, env=env, capture_output=True, text=True,
                          timeout=timeout)


def _line(out):
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.timeout(300)
def test_gpus_2_relaunches_two_ranks_and_reduces():
    r = _run(["--gpus", "2", "--dry-run", "--steps", "3", "--warmup", "1", "--no-cpu"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["gpus_active"] == 2
    assert [x["rank"] for x in d["devices"]] == [0, 1]
    assert d["dry_run"] is True
    assert d["gpu_launches"] == 2 * 3  # SUM over ranks: one stand-in launch per step per rank
    ops = d["ops"]
    assert set(ops) == {"cfg0_gray_u8_1x1080p", "cfg1_resize_u8_64x4k", "cfg2_warp_affine_f32_32x1080p",
                        "cfg3_warp_perspective_u8_16x4k", "cfg4_resize_normalize_chw_512x1080p",
                        "f4_jpeg_decode_preprocess_64x1080p"}
    for name, o in ops.items():
        assert o["verified"] is True
        assert "e2e" in o and o["ms_per_step"] > 0
    # whole-job value, weak scaling: 64 images per rank, all ranks' images
    # over the MAX time (dry ops: 1000 px per image)
    head = ops["cfg1_resize_u8_64x4k"]
    assert d["scaling"] == "weak" and d["config"]["global_batch"] == 2 * 64
    assert d["value"] == pytest.approx(2 * 64 * 1000 / (head["ms_per_step"] / 1e3) / 1e6)
    # replicas (cfg0): each rank's frames count
    g = ops["cfg0_gray_u8_1x1080p"]
    assert g["dst_mps"] == pytest.approx(2 * 1000 / (g["ms_per_step"] / 1e3) / 1e6)


@pytest.mark.timeout(120)
def test_world_size_must_match_gpus():
    r = _run(["--gpus", "2", "--dry-run", "--steps", "1", "--warmup", "1", "--no-cpu"],
             env_extra={"WORLD_SIZE": "1", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0
    assert "WORLD_SIZE=1" in r.stderr


@pytest.mark.timeout(300)
def test_reference_arm_rank0_only_under_torchrun():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "0", BENCH, "--impl", "reference", "--gpus", "2", "--dry-run",
           "--steps", "2", "--warmup", "1", "--cpu-cores", "2"]
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["impl"] == "reference" and d["cpu_baseline"]["cores"] == 2
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.timeout(300)
def test_single_rank_dry_run_carries_cpu_baseline():
    r = _run(["--dry-run", "--steps", "2", "--warmup", "1", "--cpu-cores", "2", "--ops", "resize,persp"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 1
    cb = d["cpu_baseline"]
    assert cb["cores"] == 2 and cb["value"] > 0 and cb["value_1core"] > 0
    for o in d["ops"].values():
        assert o["cpu_baseline"]["cores"] == 2
