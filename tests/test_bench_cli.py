"""CPU checks of bench.py's launch and reference-arm contracts (no GPU):

* `--gpus 2` outside torchrun relaunches itself under torch.distributed.run
  with two ranks; `--dry-run` runs the sharding and the barrier / max-over-
  ranks protocol over gloo, and the two ranks' column shards partition C4;
* the reference arm (`--impl reference`) times the compiled reference and
  never maps the product library (its inputs come from the oracle's
  generator), and prints the same `config` object as our arm.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out
    return json.loads(lines[-1])


def test_gpus_2_dry_run_two_ranks():
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--dry-run"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _last_json(r.stdout)
    assert d["dry_run"] and d["n_gpus"] == 2
    ranks = sorted(d["ranks"], key=lambda q: q["rank"])
    assert [q["rank"] for q in ranks] == [0, 1]
    assert ranks[0]["pid"] != ranks[1]["pid"]
    (a0, c0), (a1, c1) = ranks[0]["columns"], ranks[1]["columns"]
    assert a0 == 0 and a1 == c0 and c0 + c1 == 65536
    assert d["config"]["parallelism"] == "column shards x2, no collective"


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libfastleg_ref.so")),
                    reason="oracle/_ref not built")
def test_reference_arm_does_not_load_the_product():
    code = ("import sys; sys.argv = ['bench.py', '--impl', 'reference', '--cols', '2', '--steps', '1', "
            "'--warmup', '0']; import bench; bench.main(); "
            "maps = open('/proc/self/maps').read(); "
            "print('PRODUCT_LOADED', 'libfastleg_b200' in maps, 'REF_LOADED', 'libfastleg_ref' in maps)")
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert "PRODUCT_LOADED False REF_LOADED True" in r.stdout, r.stdout
    d = _last_json(r.stdout.split("PRODUCT_LOADED")[0])
    assert d["impl"] == "reference" and d["value"] > 0
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.config_dict("c4", 1, 2)
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["kind"] == "reference"
