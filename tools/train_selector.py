#!/usr/bin/env python
"""Train the learned algorithm selector from tools/selector_data.py
timings and export it as the C++ decision tree libconv2d.so evaluates (conv2d_predict, include/conv2d.h).

    python tools/train_selector.py profiles/data/selector_data_r1.json \\
        --header paper_1904_04174_b200/csrc/selector_tree.h --report profiles/data/selector_model_r1.json

Candidates = algorithms, and for implicit_gemm / matmul_1x1 each parameter variant.
Features = shape quantities the library computes from conv2d_params_t (selector_features() in api.cpp must
match FEATURES here, in order).  Model = one multi-output CART regression tree (scikit-learn) of every
candidate's log2(time / fastest time); the selector takes the supported candidate of least predicted
log-regret.  Depth chosen by 5-fold cross-validated *regret* -- time of the chosen candidate / time of the
fastest -- which is what a selector costs.
"""
from __future__ import annotations

import argparse
import json
import math

import numpy as np

try:  # the paper's layer tuples (optional: only for --paper-weight)
    import os as _os
    import sys as _sys
    _sys.path.insert(0, _os.path.dirname(_os.path.dirname(_os.path.abspath(__file__))))
    from paper_1904_04174_b200 import layers as _L
    PAPER_LAYERS = _L.RESNET50_SETS + [v for v, _ in _L.VGG16_LAYERS]
except Exception:  # pragma: no cover
    PAPER_LAYERS = []

FEATURES = ["log2_M", "log2_F", "log2_C", "log2_K2C", "window", "stride", "valid", "log2_N", "log2_HoWo",
            "tf32", "log2_pair_tiles", "log2_flops", "intensity"]


def out_hw(h, k, s, valid):
    return (h - k) // s + 1 if valid else -(-h // s)


def features(sp):
    n, h, w, c, f = sp["batch"], sp["in_rows"], sp["in_cols"], sp["channels"], sp["features"]
    k, s, valid = sp["window_rows"], sp["stride_rows"], sp["padding"]
    ho, wo = out_hw(h, k, s, valid), out_hw(w, sp["window_cols"], sp["stride_cols"], valid)
    m = n * ho * wo
    kk = k * sp["window_cols"] * c
    bn = 64 if f <= 64 else 128 if f <= 128 else 256
    tiles = math.ceil(m / 256) * math.ceil(f / bn)
    flops = 2.0 * m * f * kk
    nbytes = 4.0 * (n * h * w * c + kk * f + m * f)
    return [math.log2(m), math.log2(f), math.log2(c), math.log2(kk), k, s, valid, math.log2(n),
            math.log2(ho * wo), sp["math"], math.log2(tiles), math.log2(flops), flops / nbytes]


def c4_eligible(sp):
    """3x3 / stride 1, C <= 4, W*C % 4 == 0, F <= 128: the shapes round 2's 4-channel halo path took over."""
    return (sp["window_rows"] == 3 and sp["window_cols"] == 3 and sp["stride_rows"] == 1 and sp["stride_cols"] == 1
            and sp["channels"] <= 4 and (sp["in_cols"] * sp["channels"]) % 4 == 0 and sp["features"] <= 128)


SUPERSEDE = {"c4": c4_eligible}


def load(paths):
    """Rows of every data file, in order.  A file whose top level carries "supersedes": <class> (a re-timing of
    the shapes whose candidates changed meaning, tools/selector_data.py --replay --only <class>) first drops the
    earlier rows of that class."""
    import gzip
    rows = []
    for p in paths:
        with (gzip.open(p, "rt") if p.endswith(".gz") else open(p)) as fh:
            d = json.load(fh)
        if d.get("supersedes"):
            keep = SUPERSEDE[d["supersedes"]]
            rows = [r for r in rows if not keep(r["params"])]
        rows += d["rows"]
    return rows


def regret(rows, preds):
    out = []
    for r, c in zip(rows, preds):
        t = r["times_us"]
        best = min(t.values())
        out.append(t[c] / best if c in t else t.get("implicit_gemm/0", max(t.values())) / best)
    return np.array(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("data", nargs="+")
    ap.add_argument("--header", default="")
    ap.add_argument("--report", default="")
    ap.add_argument("--leaf", type=int, default=4, help="min samples per leaf")
    ap.add_argument("--paper-weight", type=float, default=10.0,
                    help="sample-weight factor for the paper's 35 layer tuples (b1/32/256, both maths)")
    ap.add_argument("--depth", type=int, default=0, help="fixed tree depth (skips the depth search)")
    ap.add_argument("--no-cv", action="store_true", help="fit only (no cross-validation; with --depth)")
    args = ap.parse_args()
    from sklearn.model_selection import KFold
    from sklearn.tree import DecisionTreeRegressor

    rows = load(args.data)
    X = np.array([features(r["params"]) for r in rows])
    # target: per candidate class, log2(time / fastest time) of that shape (unsupported candidates: a large
    # penalty); a multi-output regression tree averages these vectors per leaf, and the selector takes the
    # supported class of least mean log-regret -- so a class that was catastrophic for some shapes in a leaf
    # is not picked for its neighbours (a misclassification objective would not see the cost of an error)
    classes = sorted({c for r in rows for c in r["times_us"]})
    PEN = 6.0
    Y = np.array([[math.log2(r["times_us"][c] / min(r["times_us"].values())) if c in r["times_us"] else PEN
                   for c in classes] for r in rows])

    def pick(pred_row, r):
        order = np.argsort(pred_row)
        for k in order:
            if classes[k] in r["times_us"]:  # supported for this shape (the library checks conv2d_supports)
                return classes[k]
        return "implicit_gemm/0"

    # sample weight = the shape's fastest time: a selector's cost inside a network is time, so expensive
    # shapes count more; "total" regret = sum of chosen times / sum of fastest times
    tbest = np.array([min(r["times_us"].values()) for r in rows])
    wts = tbest / tbest.mean()
    if args.paper_weight != 1.0:  # the paper's layer tuples (the workload the library is benchmarked on) count more
        paper = {tuple(sorted(dict(l.params(b), math=m_).items())) for l in PAPER_LAYERS for b in (1, 32, 256)
                 for m_ in (0, 1)}
        wts = wts * np.array([args.paper_weight if tuple(sorted(r["params"].items())) in paper else 1.0 for r in rows])
    kf = KFold(5, shuffle=True, random_state=0)
    cv = {}
    # depth <= 12 keeps the compiled table well under 1 MB (depth 16 is ~4x the nodes for ~0.5% less regret)
    for depth in ((args.depth,) if args.depth else (4, 6, 8, 10, 12)):
        regs = np.ones(len(rows))
        for tr, te in ([] if args.no_cv else kf.split(X)):
            m = DecisionTreeRegressor(max_depth=depth, min_samples_leaf=args.leaf, random_state=0).fit(
                X[tr], Y[tr], sample_weight=wts[tr])
            P = m.predict(X[te])
            regs[te] = regret([rows[i] for i in te], [pick(P[q], rows[i]) for q, i in enumerate(te)])
        total = float((regs * tbest).sum() / tbest.sum())
        cv[depth] = {"mean": float(regs.mean()), "total": total, "median": float(np.median(regs)),
                     "p90": float(np.quantile(regs, 0.9)), "max": float(regs.max()), "exact": float((regs == 1.0).mean())}
        print(f"depth {depth:2d}: CV regret total {total:.4f} mean {regs.mean():.4f} median {np.median(regs):.4f} "
              f"p90 {np.quantile(regs, 0.9):.4f} max {regs.max():.2f} exact {100 * (regs == 1.0).mean():.1f}%")
    # the shallowest depth within 0.004 of the best total CV regret (smaller table, fewer outliers)
    best_total = min(v["total"] for v in cv.values())
    depth = min(d for d in cv if cv[d]["total"] <= best_total + 0.004)
    model = DecisionTreeRegressor(max_depth=depth, min_samples_leaf=args.leaf, random_state=0).fit(X, Y, sample_weight=wts)
    P = model.predict(X)
    base = {}
    for name in ("implicit_gemm/0",):
        rb = regret(rows, [name] * len(rows))
        base[name] = {"mean": float(rb.mean()), "total": float((rb * tbest).sum() / tbest.sum())}
    report = {"samples": len(rows), "features": FEATURES, "classes": classes, "depth": depth,
              "nodes": int(model.tree_.node_count), "cv_regret": cv,
              "train_regret_mean": float(regret(rows, [pick(P[i], r) for i, r in enumerate(rows)]).mean()),
              "train_regret_total": float((regret(rows, [pick(P[i], r) for i, r in enumerate(rows)]) * tbest).sum()
                                          / tbest.sum()),
              "baseline_regret_mean": base, "data": args.data}
    print(json.dumps({k: v for k, v in report.items() if k not in ("cv_regret", "classes")}, indent=1))
    if args.report:
        with open(args.report, "w") as fh:
            json.dump(report, fh, indent=1)
    if args.header:
        t = model.tree_
        algo_id = {"direct": 1, "tiled": 2, "implicit_gemm": 3, "winograd_f2x2_3x3": 4, "matmul_1x1": 5,
                   "winograd_f4x4_3x3": 6}
        lines = ["// selector_tree.h -- GENERATED by tools/train_selector.py (do not edit): the learned algorithm",
                 "// selector (SURVEY.md §8(f) N4; PAPER.md:284-288), a CART tree over selector_features() in api.cpp.",
                 f"// {len(rows)} measured shapes ({', '.join(args.data)}); depth {depth}, {t.node_count} nodes; "
                 f"leaf {args.leaf}, paper-weight {args.paper_weight:g};",
                 f"// 5-fold CV regret (chosen time / fastest time): total {cv[depth]['total']:.4f}, "
                 f"mean {cv[depth]['mean']:.4f}, median {cv[depth]['median']:.4f}, p90 {cv[depth]['p90']:.4f}.",
                 "#pragma once", "", "namespace conv2d {", "namespace selector {", "",
                 f"constexpr int kFeatures = {len(FEATURES)};",
                 f"constexpr int kNodes = {t.node_count};"]
        feat = [int(v) for v in t.feature]
        thr = [float(v) for v in t.threshold]
        lines.append("// per node: feature (-2 = leaf), threshold (go left if x[feature] <= threshold), left, right")
        lines.append("constexpr int kFeature[kNodes] = {" + ", ".join(map(str, feat)) + "};")
        lines.append("constexpr double kThreshold[kNodes] = {" + ", ".join(f"{v:.9g}" for v in thr) + "};")
        lines.append("constexpr int kLeft[kNodes] = {" + ", ".join(str(int(v)) for v in t.children_left) + "};")
        lines.append("constexpr int kRight[kNodes] = {" + ", ".join(str(int(v)) for v in t.children_right) + "};")
        cls = classes
        lines.append(f"constexpr int kClasses = {len(cls)};")
        algos = [algo_id[c.split("/")[0]] for c in cls]
        vars_ = [int(c.split("/")[1]) if "/" in c else 0 for c in cls]
        lines.append("// class -> (conv2d_algo_t, variant): " + ", ".join(cls))
        lines.append("constexpr int kClassAlgo[kClasses] = {" + ", ".join(map(str, algos)) + "};")
        lines.append("constexpr int kClassVariant[kClasses] = {" + ", ".join(map(str, vars_)) + "};")
        leaves = [nd for nd in range(t.node_count) if t.children_left[nd] < 0]
        leaf_of = {nd: i for i, nd in enumerate(leaves)}
        lines.append(f"constexpr int kLeaves = {len(leaves)};")
        lines.append("// per node: its row in kLogRegret if it is a leaf, else -1")
        lines.append("constexpr int kLeafRow[kNodes] = {" +
                     ", ".join(str(leaf_of.get(nd, -1)) for nd in range(t.node_count)) + "};")
        lines.append("// per leaf: mean log2(time / fastest) of each class over the training shapes that reach it")
        vals = []
        for nd in leaves:
            vals.append("{" + ", ".join(f"{float(v):#.3g}f" for v in t.value[nd][:, 0]) + "}")
        lines.append("constexpr float kLogRegret[kLeaves][kClasses] = {\n" + ",\n".join(vals) + "};")
        lines += ["", "}  // namespace selector", "}  // namespace conv2d", ""]
        with open(args.header, "w") as fh:
            fh.write("\n".join(lines))


if __name__ == "__main__":
    main()
