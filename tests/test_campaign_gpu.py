"""run_campaign (bench.hpp:382-524) through the drop-in: ONE program written against the reference's
bench.hpp API (examples/campaign_example.cpp) is compiled against the unmodified reference headers
(oracle/_ref/campaign_ref, CPU) and against include/hpclust/bench.hpp over libhpcg.so
(examples/campaign_example, GPU); the two campaigns must agree series by series."""
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
EXE = ROOT / "examples" / "campaign_example"
REF = ROOT / "oracle" / "_ref" / "campaign_ref"


def _run(exe, *args):
    out = subprocess.run([str(exe), *map(str, args)], capture_output=True, text=True, timeout=600)
    assert out.stdout, out.stderr
    r = json.loads(out.stdout)
    assert "error" not in r, r
    return r


def _need():
    if not EXE.exists():
        subprocess.run(["make", "-C", str(ROOT / "examples")], check=True)
    if not REF.exists():
        pytest.skip("reference campaign binary not built (oracle/_ref/campaign_ref)")


def test_campaign_metrics_and_blobs_equal_reference_host_only():
    # gen_blobs (bench.hpp:171-205) and the metric helpers (bench.hpp:18-135): bit-equal, no device
    _need()
    for args in [(5000, 4, 5, 0, 9, "metrics", 0), (2187, 10, 10, 0, 4, "metrics", 0), (101, 1, 7, 0, 12, "metrics", 0)]:
        assert _run(EXE, *args) == _run(REF, *args)


def _close(a, b, rel, abs_=0.0):
    if a is None or b is None:
        return a is b
    return abs(a - b) <= max(abs_, rel * max(abs(a), abs(b)))


@pytest.mark.gpu
@pytest.mark.parametrize("algos,ks", [("inner,competitive,cooperative,hybrid", "4,6"),
                                      ("competitive,hybrid,forgy,pbk", "5")])
def test_campaign_equals_reference(algos, ks):
    _need()
    args = (20000, 3, 6, 6, 3, algos, ks)
    g, e = _run(EXE, *args), _run(REF, *args)
    assert g["rows"] == e["rows"] and g["checksum"] == e["checksum"]
    assert len(g["series"]) == len(e["series"]) == len(algos.split(",")) * len(ks.split(","))
    for sg, se in zip(g["series"], e["series"]):
        tag = (se["algorithm"], se["k"])
        for key in ("dataset", "algorithm", "k", "n_d_median", "n_s_median", "sample_size", "time_limit", "t1", "t2",
                    "succ"):
            assert sg[key] == se[key], (tag, key)
        hp = se["algorithm"] not in ("forgy", "pbk")
        for rg, re_ in zip(sg["records"], se["records"]):
            assert rg["rep"] == re_["rep"] and rg["n_d"] == re_["n_d"], tag
            # epsilon = 100 (f - f*) / f*: objectives agree to 1e-12 relative, so epsilon to ~1e-9 absolute
            assert _close(rg["epsilon"], re_["epsilon"], 0.0, 1e-8), tag
            if hp:  # lockstep clock: sample counts; the baselines report wall seconds
                assert rg["t"] == re_["t"] and rg["t_bar"] == re_["t_bar"], tag
        for name in ("median", "min", "max", "stddev"):
            assert _close(sg["epsilon"][name], se["epsilon"][name], 0.0, 1e-8), (tag, name)
            if hp:
                assert sg["t"][name] == se["t"][name], (tag, name)
                assert (sg["t_bar"] is None) == (se["t_bar"] is None)
                if se["t_bar"] is not None:
                    assert sg["t_bar"][name] == se["t_bar"][name], (tag, name)
