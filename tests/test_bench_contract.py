"""bench.py keeps the driver's JSON contract: one JSON line with the required keys, on the reference arm
(CPU oracle, -m "not gpu") and on the CUDA arm (-m gpu, small step counts)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e", "cpu_baseline"}


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.strip()]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    d = _run(["--impl", "reference", "--config", "0", "--steps", "2", "--warmup", "1"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_cuda_arm_json_line():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--config", "1", "--steps", "5", "--warmup", "3", "--cpu-budget", "1", "--no-extras"])
    assert BASE_KEYS <= set(d) | {"roofline", "gpu_launches", "clocks"}
    assert {"roofline", "gpu_launches", "clocks"} <= set(d)
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.5
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["gpu_launches"] == 5 * 1  # row split: one kernel per step
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    assert d["config"]["algo"] == "rowsplit" and d["config"]["l2"].startswith("flushed")
    assert d["dtype"] == "f32" and d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3
    assert d["plan_ms"] > 0 and d["cpu_baseline"]["physical_cores"] >= 1
    assert 0 < r["ceiling"]["frac_ceiling"] <= 1.0


@pytest.mark.gpu
def test_cuda_arm_merge_config_and_extras():
    """R-MAT 22 as the head (merge: partition + compute + fix-up per step) plus the configs[1] key."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _run(["--config", "2", "--steps", "4", "--warmup", "3", "--no-cpu-baseline", "--no-e2e"])
    assert d["config"]["algo"] == "merge" and d["gpu_launches"] == 4 * 3
    assert d["roofline"]["kernel"] == "k_merge_w" and d["scaling"] == "strong"
    assert "config1" in d and d["config1"]["algo"] == "rowsplit" and d["config1"]["value"] > 0
    assert d["config1"]["roofline"]["frac"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["1", "2"])
def test_torchrun_single_rank_exercises_the_distributed_path(cfg):
    """Under torchrun (even one rank) bench.py runs the multi-GPU plumbing for real: NCCL process group,
    row-block partition + slicing, broadcast of B (timed), max-over-ranks reductions, all-gather of C
    (timed) and the e2e path with the broadcast."""
    import socket
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "1", "--config", cfg, "--steps", "3", "--warmup", "3", "--gather-c",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 0
    assert d["config"]["bcast_B_ms"] is not None and d["config"]["allgather_C_ms"] is not None
    assert "NCCL broadcast" in d["e2e"]["includes"]


def test_traffic_capture_matches_the_build_by_sources(tmp_path, monkeypatch):
    # roofline.traffic comes from profiles/ncu_traffic.json; it counts as the same build when the library
    # hash OR the source hash matches (nvcc .so files are not bit-reproducible), and never for a variant
    # library selected with SPMM_LIB unless its own hash matches
    sys.path.insert(0, ROOT)
    import bench
    from paper_1803_08601_b200 import build as B
    (tmp_path / "profiles").mkdir()
    ent = {"dram_bytes": 1, "lib_sha16": "0" * 16, "src_sha16": B.source_sha16()}
    (tmp_path / "profiles" / "ncu_traffic.json").write_text(json.dumps({"k": ent}))
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    monkeypatch.delenv("SPMM_LIB", raising=False)
    assert bench.load_traffic("k", "f" * 16)["same_build"] is True       # sources match
    assert bench.load_traffic("k", "0" * 16)["same_build"] is True       # library matches
    monkeypatch.setenv("SPMM_LIB", "/nonexistent/variant.so")
    assert bench.load_traffic("k", "f" * 16)["same_build"] is False      # a variant: hash only
    monkeypatch.delenv("SPMM_LIB")
    ent["src_sha16"] = "1" * 16
    (tmp_path / "profiles" / "ncu_traffic.json").write_text(json.dumps({"k": ent}))
    assert bench.load_traffic("k", "f" * 16)["same_build"] is False      # stale capture
