"""Generates tests/golden/configs.json (+ labels_*.npz) — run HERE, in the build container.

Inputs are the five BASELINE.json configs built by the repo's seeded synthetic generator
(SURVEY.md §8d), hashed (SHA-256) so a changed generator is caught. Outputs come from:

* the UNMODIFIED reference library (oracle/_ref/libseghdc_ref.so: /root/reference sources
  compiled with their own flags) for C0, C1 and C2 images 0-3 — its own encode_image and the
  replay of its cluster() loop through select_initial_centroids/assign_labels/update_centroids;
* the C restatement (oracle/lib/libseghdc_oracle.so), checked bit-identical to the reference on
  those same cases, for the rest of C2, for C3 (20 rounds) and for the first 2 rounds of C4
  (the full 20-round C4 run would take ~1 h on 8 cores; its 34 GB grid does not fit host memory,
  so the streaming port so_cluster_stream re-encodes each pixel every pass).

Usage: python tests/golden/make_golden.py [--only C0,C1,...]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2303_12753_b200 as S  # noqa: E402

# (config id, dim, k, iterations, alpha) — BASELINE.json configs; alpha = 1.0 for C3/C4 because
# the default 0.2 fails the reference's flip-unit validation at 2048^2 / 4096^2.
CONFIGS = {
    "C0": dict(cid=0, dim=10000, k=2, iterations=10, alpha=0.2),
    "C1": dict(cid=1, dim=10000, k=2, iterations=10, alpha=0.2),
    "C2": dict(cid=2, dim=10000, k=2, iterations=10, alpha=0.2),
    "C3": dict(cid=3, dim=10000, k=4, iterations=20, alpha=1.0),
    "C4": dict(cid=4, dim=16384, k=8, iterations=20, alpha=1.0),
}
BETA, GAMMA, CB_SEED = 26, 1, 0


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def record(img, res, iterations, seeds):
    return {
        "image_sha256": sha(img),
        "seeds": [int(s) for s in seeds],
        "iterations": iterations,
        "rounds": int(res["rounds"]),
        "labels_sha256": sha(res["labels"].astype(np.uint32)),
        "round_labels_sha256": [sha(r.astype(np.uint32)) for r in res["labels_rounds"]],
        "round_counts": [np.bincount(r, minlength=res["centroids"].shape[0]).tolist() for r in res["labels_rounds"]],
        "centroids_sha256": sha(res["centroids"].astype(np.uint32)),
        "counts": [int(x) for x in res["counts"]],
    }


def run_case(name, spec, image_seed, use_ref, iterations=None, early_stop=False, stream=False):
    P = oracle.Port()
    img = S.synth_image(spec["cid"], image_seed)
    h, w, c = img.shape
    it = iterations or spec["iterations"]
    row, col, wid = S.build_codebooks(spec["dim"], h, w, c, spec["alpha"], BETA, GAMMA, CB_SEED)
    seeds = P.select_seeds(img, spec["k"])
    t = time.time()
    if stream:  # the grid does not fit host memory (C4: 34 GB): re-encode every pass
        grid = None
        res = P.cluster_stream(img, spec["dim"], row, col, wid, spec["k"], it, early_stop, per_round=True)
    else:
        grid = P.encode(img, spec["dim"], row, col, wid)
        res = P.cluster(grid, img, spec["dim"], spec["k"], it, early_stop, per_round=True)
    out = record(img, res, it, seeds)
    out["port_seconds"] = round(time.time() - t, 2)
    if grid is not None:
        out["grid_sha256"] = sha(grid)
    if use_ref:
        R = oracle.Ref()
        rgrid = R.encode(img, spec["dim"], spec["alpha"], BETA, GAMMA, CB_SEED)
        assert (rgrid == grid).all(), f"{name}: port encode != reference encode_image"
        rseeds = R.select_seeds(img, spec["k"])
        assert (rseeds == seeds).all(), f"{name}: seeds differ"
        t = time.time()
        rres = R.cluster_replay(rgrid, img, spec["dim"], spec["k"], it, early_stop, per_round=True)
        real = R.cluster(rgrid, img, spec["dim"], spec["k"], it, early_stop, per_round=True)
        rec = record(img, rres, it, rseeds)
        assert (real["labels_rounds"] == rres["labels_rounds"]).all(), f"{name}: replay != cluster()"
        for key in ("labels_sha256", "round_labels_sha256", "centroids_sha256", "counts", "rounds"):
            assert rec[key] == out[key], f"{name}: port disagrees with the reference on {key}"
        out["ref_seconds"] = round(time.time() - t, 2)
        out["source"] = "reference (oracle/_ref) == port"
    else:
        out["source"] = "port (oracle/lib), validated against the reference on C0/C1/C2[0:4]"
    return out, res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C0,C1,C2,C3,C4")
    args = ap.parse_args()
    oracle.build()
    path = os.path.join(HERE, "configs.json")
    data = json.load(open(path)) if os.path.exists(path) else {}
    data["_meta"] = {"beta": BETA, "gamma": GAMMA, "codebook_seed": CB_SEED, "generator": "tests/golden/make_golden.py",
                     "configs": CONFIGS}
    only = args.only.split(",")
    for name in only:
        spec = CONFIGS[name]
        t0 = time.time()
        if name in ("C0", "C1"):
            rec, res = run_case(name, spec, 0, use_ref=True)
            es, _ = run_case(name, spec, 0, use_ref=True, early_stop=True)
            rec["early_stop_rounds"] = es["rounds"]
            rec["early_stop_labels_sha256"] = es["labels_sha256"]
            np.savez_compressed(os.path.join(HERE, f"labels_{name}.npz"), labels=res["labels"].astype(np.uint8),
                                centroids=res["centroids"])
            data[name] = rec
        elif name == "C2":
            imgs = []
            for s in range(64):
                rec, _ = run_case(name, spec, s, use_ref=s < 4)
                imgs.append(rec)
            data[name] = {"images": imgs}
        elif name == "C3":
            rec, _ = run_case(name, spec, 0, use_ref=False)
            data[name] = rec
        elif name == "C4":
            rec, _ = run_case(name, spec, 0, use_ref=False, iterations=2, stream=True)
            rec["source"] = ("port (oracle/lib so_cluster_stream: pixels re-encoded every pass), first 2 rounds; "
                             "so_cluster_stream == so_cluster is pinned by tests/test_oracle.py")
            data[name] = rec
        print(f"{name}: {time.time() - t0:.1f}s", flush=True)
        json.dump(data, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
