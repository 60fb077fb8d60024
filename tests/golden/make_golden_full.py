"""Full-length C3 / C4 goldens from the UNMODIFIED reference (run HERE, in the build container).

Writes the C3 (2048^2 x 3, D = 10000, K = 4, 20 rounds) and C4 (4096^2 x 3, D = 16384, K = 8,
20 rounds) records of tests/golden/configs.json:

* labels of every round, the centroid set used by the final assignment and its member counts
  come from the reference's own encode_image / assign_labels / update_centroids
  (oracle/_ref ``ref_pare_*``: row-block shards, each encoded by the reference's encode_image,
  assign + update per shard on its own thread, integer sums combined exactly; the loop is
  cluster()'s, clusterer.cpp:190-218, early stop off as in the reference's bench);
* the per-round count of strictly_closer comparisons whose unsigned __int128 products wrap
  (clusterer.cpp:41-50) comes from the C restatement's streaming loop (so_cluster_stream +
  so_last_wraps), which must agree with the reference on every round's labels first.

C4 needs ~35 GB of host memory for the reference's grid and about an hour on 8 cores.

Usage: python tests/golden/make_golden_full.py [--only C3,C4]
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
import workloads  # noqa: E402

NAMES = {"C3": 3, "C4": 4}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run(name: str) -> dict:
    spec = workloads.CONFIGS[NAMES[name]]
    img = workloads.synth_image(spec["cid"], 0)
    h, w, c = img.shape
    dim, k, it, alpha = spec["dim"], spec["k"], spec["iterations"], spec["alpha"]
    R, P = oracle.Ref(), oracle.Port()
    t0 = time.time()
    round_hash, round_counts = [], []

    def on_round(r, labels):
        round_hash.append(sha(labels))
        round_counts.append(np.bincount(labels, minlength=k).tolist())
        print(f"  {name} reference round {r}: {time.time() - t0:.0f}s counts {round_counts[-1]}", flush=True)

    res = R.cluster_encoded(img, dim, k, it, alpha=alpha, beta=workloads.BETA, gamma=workloads.GAMMA,
                            seed=workloads.CB_SEED, on_round=on_round)
    ref_s = time.time() - t0
    rec = {
        "image_sha256": sha(img),
        "seeds": [int(s) for s in res["seeds"]],
        "iterations": it,
        "rounds": it,
        "labels_sha256": round_hash[-1],
        "round_labels_sha256": round_hash,
        "round_counts": round_counts,
        "centroids_sha256": sha(res["centroids"].astype(np.uint32)),
        "counts": [int(x) for x in res["counts"]],
        "ref_seconds": round(ref_s, 1),
    }
    del res
    # the restatement's streaming loop: same labels every round, plus the 128-bit wrap counts
    row, col, wid = P.build_codebooks(dim, h, w, c, alpha, workloads.BETA, workloads.GAMMA, workloads.CB_SEED)
    t1 = time.time()
    pres = P.cluster_stream(img, dim, row, col, wid, k, it, False, per_round=True)
    wraps = P.last_wraps()
    port_hash = [sha(x.astype(np.uint32)) for x in pres["labels_rounds"]]
    assert port_hash == round_hash, f"{name}: port labels differ from the reference"
    assert sha(pres["centroids"].astype(np.uint32)) == rec["centroids_sha256"], f"{name}: port centroids differ"
    assert [int(x) for x in pres["counts"]] == rec["counts"], f"{name}: port counts differ"
    rec["round_wraps"] = wraps
    rec["port_seconds"] = round(time.time() - t1, 1)
    rec["source"] = ("reference (oracle/_ref: encode_image/assign_labels/update_centroids, row shards on threads, "
                     "all rounds) == port so_cluster_stream (which also counts 128-bit comparator wraps)")
    print(f"{name}: reference {ref_s:.0f}s, port {rec['port_seconds']}s, wraps {wraps}", flush=True)
    return rec


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="C3,C4")
    args = ap.parse_args()
    oracle.build()
    path = os.path.join(HERE, "configs.json")
    for name in args.only.split(","):
        rec = run(name)
        data = json.load(open(path))  # re-read: other records may have changed meanwhile
        data[name] = rec
        json.dump(data, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
