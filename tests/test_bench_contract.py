"""The bench.py contract pieces that run without a GPU: the reference arm's
JSON line (the oracle on a bounded sample of the default workload, C3) and the host helpers the
GPU arm's line is built from (slab split, occupied cells, peaks)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "2",
                          "--warmup", "1", "--ref-sample", "4000"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["n_gpus"] == 1 and line["steps"] == 2
    assert line["value"] > 0 and line["higher_is_better"] is True and line["dtype"] == "f64"
    assert line["config"]["workload"] == "C3"   # the N = 1 default: largest single-GPU config
    assert line["cpu_baseline"]["host"]["nproc"] >= 1
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": line["unit"], "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}


def test_host_helpers():
    import bench
    from synth import get_config
    wl = get_config("C2")
    assert bench.slab_split(wl, 1) == [0, wl.nz]
    assert bench.occupied_cells(wl, 0, wl.nz) == wl.nx * wl.ny * wl.nz
    c5 = get_config("C5")
    split = bench.slab_split(c5, 8)
    assert split[0] == 0 and split[-1] == c5.nz and len(split) == 9
    assert all(b > a for a, b in zip(split, split[1:]))
    # occupied cells of the C5 plasma slab (z in [600, 700)) only
    assert sum(bench.occupied_cells(c5, a, b) for a, b in zip(split, split[1:])) == c5.nx * c5.ny * 100
    peak, src = bench.load_peaks()
    assert peak > 1000 and isinstance(src, str)
    tf, tsrc = bench.load_fp64_peak()
    assert 10 < tf < 100 and isinstance(tsrc, str)
    roof = bench.fp64_roof(20e9, None, {}, tf, tsrc)
    assert roof["frac"] is None and roof["paper_flop_per_update"] == 336.0
    roof = bench.fp64_roof(20e9, 250.0, {"commit": "abc"}, tf, tsrc)
    assert roof["frac"] == pytest.approx(20e9 * 250.0 / 1e12 / tf)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_weak_scaling_workload_per_rank(world):
    from synth import get_config
    wl = get_config("C4").for_ranks(world)
    assert wl.nz == 128 * world and wl.nx == wl.ny == 256
