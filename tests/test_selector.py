"""Learned selector (include/conv2d.h conv2d_predict) -- host-side, no GPU.

* The C++ tree walk (api.cpp selector_features / selector_predict) equals a Python walk of the exported
  tree (paper_1904_04174_b200/csrc/selector_tree.h) driven by the training script's own feature code
  (tools/train_selector.py FEATURES), on the measured shapes and on random ones -- so the two feature
  definitions cannot drift apart.
* Every prediction is a candidate the library can run for those params (algorithm supported, variant
  enumerated).
* Replayed over the measured data (profiles/data/selector_data_r1*.json), the predictions cost at most a few
  percent over the per-shape fastest candidate, far below always taking implicit_gemm/0.
"""
import importlib.util
import json
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "paper_1904_04174_b200", "csrc", "selector_tree.h")
DATA = [os.path.join(ROOT, "profiles", "data", f)
        for f in ("selector_data_r1.json", "selector_data_r1b.json", "selector_data_r1c.json", "selector_data_r1d.json.gz",
                  "selector_data_r2_c4.json")]  # r2_c4: the C <= 4 3x3 shapes re-timed on the 4-channel halo path


@pytest.fixture(scope="module")
def C():
    from paper_1904_04174_b200 import conv2d
    return conv2d


@pytest.fixture(scope="module")
def tree():
    src = open(HEADER).read()

    def arr(name, conv):
        m = re.search(r"constexpr \w+ " + name + r"\[[^\]]*\](?:\[[^\]]*\])? = \{(.*?)\};", src, re.S)
        body = m.group(1).replace("{", "").replace("}", "").replace("f", "")
        return [conv(v) for v in body.split(",") if v.strip()]
    t = {k: arr(k, int) for k in ("kFeature", "kLeft", "kRight", "kLeafRow", "kClassAlgo", "kClassVariant")}
    t["kThreshold"] = arr("kThreshold", float)
    ncls = len(t["kClassAlgo"])
    flat = arr("kLogRegret", float)
    t["kLogRegret"] = np.array(flat, dtype=np.float32).reshape(-1, ncls)
    return t


@pytest.fixture(scope="module")
def feats():
    spec = importlib.util.spec_from_file_location("train_selector", os.path.join(ROOT, "tools", "train_selector.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m.features


def enumerated(C, p, a, v):
    if a not in (C.ALGO_IMPLICIT_GEMM, C.ALGO_MATMUL_1X1):
        return v == 0
    old = C.conv2d_get_variant(p, a)
    try:
        C.conv2d_set_variant(p, a, v)
        ok = True
    except C.Conv2dError:
        ok = False
    C.conv2d_set_variant(p, a, old)
    return ok


def py_predict(C, tree, feats, sp):
    x = np.array(feats(sp))
    node = 0
    while tree["kFeature"][node] >= 0:
        f = tree["kFeature"][node]
        node = tree["kLeft"][node] if x[f] <= tree["kThreshold"][node] else tree["kRight"][node]
    lr = tree["kLogRegret"][tree["kLeafRow"][node]]
    p = C.Params(**sp)
    for k in np.argsort(lr, kind="stable"):
        a, v = tree["kClassAlgo"][k], tree["kClassVariant"][k]
        if C.conv2d_supports(p, a) and enumerated(C, p, a, v):
            return a, v
    return C.ALGO_IMPLICIT_GEMM, 0


def random_params(rng, n):
    out = []
    while len(out) < n:
        k = int(rng.choice([1, 2, 3, 5, 7]))
        s = int(rng.choice([1, 2, 3]))
        h = int(rng.integers(k, 240))
        sp = dict(batch=int(rng.choice([1, 3, 16, 64, 256])), in_rows=h, in_cols=int(rng.integers(k, 240)),
                  channels=int(rng.integers(1, 1200)), features=int(rng.integers(1, 1200)), window_rows=k,
                  window_cols=k, stride_rows=s, stride_cols=s, padding=int(rng.integers(0, 2)),
                  math=int(rng.integers(0, 2)))
        out.append(sp)
    return out


def test_cpp_walk_equals_python_walk(C, tree, feats):
    rows = json.load(open(DATA[0]))["rows"][:400]
    shapes = [r["params"] for r in rows] + random_params(np.random.default_rng(5), 400)
    for sp in shapes:
        assert C.conv2d_predict(C.Params(**sp)) == py_predict(C, tree, feats, sp), sp


def test_predictions_are_runnable(C):
    for sp in random_params(np.random.default_rng(6), 300):
        p = C.Params(**sp)
        a, v = C.conv2d_predict(p)
        assert C.conv2d_supports(p, a), sp
        assert enumerated(C, p, a, v), (sp, a, v)


def test_replayed_regret_on_measured_shapes(C):
    chosen, fastest, base = [], [], []
    import gzip
    for path in DATA:
        with (gzip.open(path, "rt") if path.endswith(".gz") else open(path)) as fh:
            data = json.load(fh)
        for r in data["rows"]:
            t = r["times_us"]
            a, v = C.conv2d_predict(C.Params(**r["params"]))
            name = C.ALGO_NAMES[a] + (f"/{v}" if a in (C.ALGO_IMPLICIT_GEMM, C.ALGO_MATMUL_1X1) else "")
            assert name in t, (r["params"], name)
            chosen.append(t[name])
            fastest.append(min(t.values()))
            base.append(t["implicit_gemm/0"])
    chosen, fastest, base = map(np.array, (chosen, fastest, base))
    total = chosen.sum() / fastest.sum()
    assert total < 1.03, total                      # training-set total time within 3% of the per-shape best
    assert np.mean(chosen / fastest) < 1.04
    assert total < base.sum() / fastest.sum() - 0.1  # far better than always implicit_gemm/0 (~1.18)


def test_auto_policy_validation(C):
    with pytest.raises(C.Conv2dError):
        C.conv2d_set_auto_policy(7)
    for pol in (C.AUTO_PREDICT, C.AUTO_HYBRID, C.AUTO_MEASURE):
        C.conv2d_set_auto_policy(pol)


def test_committed_tree_is_reproducible_from_committed_data(tmp_path):
    """selector_tree.h is exactly what tools/train_selector.py fits to profiles/data/selector_data_r1*.json (the
    depth the committed header states, no cross-validation needed): the compiled model has a provenance."""
    import subprocess
    import sys
    src = open(HEADER).read()
    m = re.search(r"depth (\d+), \d+ nodes; leaf (\d+), paper-weight ([0-9.]+)", src)
    out = tmp_path / "tree.h"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "train_selector.py"), *DATA, "--depth", m.group(1),
                        "--leaf", m.group(2), "--paper-weight", m.group(3), "--no-cv", "--header", str(out)],
                       capture_output=True, text=True, cwd=ROOT)
    assert r.returncode == 0, r.stderr
    strip = lambda s: "\n".join(l for l in s.splitlines() if not l.startswith("//"))  # noqa: E731
    assert strip(out.read_text()) == strip(src)
