"""bench.py's JSON contract, on one GPU: the N=1 line and the N>1 (slab-decomposed) line.

The N>1 run here puts both torchrun ranks on GPU 0 with gloo (SPH_BENCH_SHARE_GPU=1), which
exercises the decomposed path (DeviceSlabSim: migration, halo, rho refresh) and the JSON
fields; its timings mean nothing."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
            "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
            "gpu_launches", "clocks"]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _last_json(out):
    return json.loads([l for l in out.splitlines() if l.startswith("{")][-1])


@pytest.mark.gpu
def test_bench_single_gpu_line():
    out = subprocess.run([sys.executable, "bench.py", "--particles", "65536", "--steps", "3",
                          "--warmup", "3", "--e2e-steps", "2", "--cpu-baseline", "0"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600, check=True).stdout
    d = _last_json(out)
    for k in REQUIRED + ["roofline", "roofline_step"]:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 65536 * 272


@pytest.mark.gpu
def test_bench_decomposed_two_ranks_on_one_gpu():
    env = dict(os.environ, SPH_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--particles", "65536", "--steps", "2", "--warmup", "3", "--e2e-steps", "1"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900,
                         check=True).stdout
    d = _last_json(out)
    for k in REQUIRED:
        assert k in d, k
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert "slab decomposition" in d["config"]["parallelism"]
    assert d["config"]["n"] == 2 * 65536
    assert d["exchange_bytes_per_step_rank0"] > 0


def test_reference_arm_is_the_reference_on_cpu(ref):
    """--impl reference: full reference steps (every cell), nothing of libsph_b200 loaded."""
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--particles", "20000",
                          "--ppc", "64", "--steps", "2", "--warmup", "1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600, check=True).stdout
    d = _last_json(out)
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["gpu_launches"] == 0
    assert "every cell" in d["cpu_baseline"]["sample"]
    assert not any("libsph_b200" in p for p in d["native_libs_loaded"])
    assert "oracle/_ref/libsoaview_ref.so" in d["native_libs_loaded"]
