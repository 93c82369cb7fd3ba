"""bench.py's contract.

CPU: the reference arm (`--impl reference`) never loads the product package
or its library, prints the GPU arm's static config keys and the steps it
really timed.  GPU: the N>1 path from one process (slabs sharing the visible
devices) prints a line with parity, e2e, roofline and comm fields.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_PROBE = r"""
import json, runpy, sys
sys.argv = ["bench.py"] + sys.argv[1:]
runpy.run_path("bench.py", run_name="__main__")
loaded = sorted(m for m in sys.modules if m.startswith("paper_2303_08365_b200"))
maps = open("/proc/self/maps").read()
print(json.dumps({"probe": True, "product_modules": loaded,
                  "product_so": "libtessera_b200" in maps}))
"""


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, "-c", _PROBE] + args, cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    return lines


def test_reference_arm_is_product_free():
    import oracle
    if not oracle.Reference.available():
        pytest.skip("reference library not built (oracle/_ref)")
    line, probe = _run(["--impl", "reference", "--config", "c3", "--steps", "3",
                        "--warmup", "3"])
    assert probe["product_modules"] == [] and not probe["product_so"]
    assert line["impl"] == "reference"
    # K rounded up to whole tb=10 rounds of run_tessellated, reported as such
    assert line["steps"] == 10 and line["steps_requested"] == 3
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0

    sys.path.insert(0, ROOT)
    import bench
    assert line["config"] == bench.bench_config(bench.CONFIGS["c3"], 1)
    assert line["metric"] == bench.METRIC


def test_config_is_static_and_scales():
    sys.path.insert(0, ROOT)
    import bench
    c3 = bench.bench_config(bench.CONFIGS["c3"], 4)
    assert c3["extent_per_gpu"] == [512, 512, 512]
    assert c3["global_extent"] == [2048, 512, 512] and c3["parallelism"] == "slab4"
    c4 = bench.bench_config(bench.CONFIGS["c4"], 8)
    assert c4["extent_per_gpu"] == [128, 1024, 1024] and c4["global_extent"] == [1024] * 3
    assert bench.cfg_scaling(bench.CONFIGS["c4"]) == "strong"


@pytest.mark.gpu
def test_bench_two_slabs_from_one_process():
    line, _ = _run(["--gpus", "2", "--share-devices", "--config", "c3", "--steps", "6",
                    "--warmup", "3", "--no-cpu"], timeout=900)
    assert line["n_gpus"] == 2 and line["scaling"] == "weak"
    assert line["config"]["global_extent"] == [1024, 512, 512]
    assert line["parity"]["checked"] and line["parity"]["bitwise_equal"], line["parity"]
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0
    assert line["comm"]["messages"] > 0 and line["gpu_launches"] > 0
    assert line["roofline"]["frac"] > 0
