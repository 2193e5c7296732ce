"""C3 (BASELINE configs[2]): the ogbn-mag-shaped synthetic graph (C2's),
2-layer RGAT with 4 heads (hidden 64, fanout [25,20], batch 1024) on one B200, with
the partition-aware cache accounting at 10/25/50% of the layer-0 feature rows
(presample_hotness -> fill_and_serve top-k, cache.cpp:39-141; hits and misses of
every step's layer-0 frontier, harness.cpp:425-437).

    python tools/bench_c3.py [--steps 20] [--warmup 3] [--fracs 0.1,0.25,0.5] [--out f.json]

Prints one JSON object: device-resident and end-to-end sampled edges/s, per-class
device time, and the hit rates per cache capacity (RGCN on the same batches beside
it for reference)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_09697_b200 import hetsim as H  # noqa: E402

SEED = 1
FANOUTS = [25, 20]


def run(g, batches, seeds, args, model, cache_ids=None):
    eng = H.Engine.for_experiment(g, FANOUTS, 64, SEED, batch_cap=1024, model=model, heads=4)
    eng.set_option("retain_grads", 0)
    if cache_ids is not None:
        eng.set_cache(cache_ids)
    w, k = args.warmup, args.steps
    eng.bench(batches[:w], seeds[:w])
    ms, _, loss = eng.bench(batches[w:w + k], seeds[w:w + k])
    edges = 0
    for b, s in zip(batches[w:w + k], seeds[w:w + k]):
        eng.sample(b, s)
        edges += int(eng.read("sampled_edges")["sampled_edges"][0])
    out = {"value": edges / (ms / 1000.0), "ms_per_step": ms / k, "sampled_edges_per_step": edges / k,
           "final_loss": loss}
    eng.profile(True)
    eng.bench(batches[w:w + min(k, 10)], seeds[w:w + min(k, 10)])
    prof = eng.profile_read()
    eng.profile(False)
    out["kernel_us_per_step"] = {kk.split(".")[1]: round(float(v[0]) * 1000.0 / min(k, 10), 1)
                                 for kk, v in sorted(prof.items()) if kk.endswith(".ms")}
    te = time.perf_counter()
    e_edges = 0
    eb, es = batches[w + k:w + 2 * k], seeds[w + k:w + 2 * k]
    eng.prefetch(eb[0], es[0])
    for i, (b, s) in enumerate(zip(eb, es)):
        if i + 1 < len(eb):
            eng.prefetch(eb[i + 1], es[i + 1])
        e_edges += eng.step(b, s)["sampled_edges"]
    out["e2e"] = e_edges / (time.perf_counter() - te)
    if cache_ids is not None:
        out["cache_counters"] = {kk: v.tolist() for kk, v in eng.cache_counters().items()}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--fracs", default="0.1,0.25,0.5")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    spec = H.ogbn_mag_spec()
    g = H.gen_synthetic(spec, SEED)
    need = args.warmup + 2 * args.steps + 2
    batches = H.make_batches(g, 1024, need, H.mix_seed(SEED, 0xBA7C))
    seeds = [H.mix_seed(SEED, 0xB000 + i) for i in range(len(batches))]
    res = {"workload": "C3 (BASELINE configs[2]): ogbn-mag-shaped synthetic, 2-layer RGAT 4 heads, hidden 64, "
                       "fanout [25,20], batch 1024, 1 B200, f32 tables",
           "metric": "sampled-edges/s", "data": "synthetic"}
    res["rgat"] = run(g, batches, seeds, args, "rgat")
    res["rgcn_same_batches"] = run(g, batches, seeds, args, "rgcn")
    # hotness of one presample epoch, then the static top-k fill per capacity fraction
    eng = H.Engine.for_experiment(g, FANOUTS, 64, SEED, batch_cap=1024)
    hot = eng.presample_hotness(1, H.mix_seed(SEED, 0xCA11E), 1024)
    del eng
    res["cache"] = {}
    for frac in [float(x) for x in args.fracs.split(",") if x]:
        cached = []
        for t in range(len(spec["node_types"])):
            counts = hot.get(f"hot.t{t}")
            if counts is None or len(counts) == 0:
                cached.append(np.zeros(0, np.uint32))
                continue
            cap = int(frac * len(counts))
            order = np.lexsort((np.arange(len(counts)), -counts.astype(np.int64)))[:cap]
            cached.append(np.sort(order).astype(np.uint32))
        r = run(g, batches, seeds, args, "rgat", cache_ids=cached)
        stats = {}
        for kk, v in r.pop("cache_counters").items():
            hits, misses = int(v[0]), int(v[1])
            stats[kk] = {"hits": hits, "misses": misses, "hit_rate": round(hits / max(1, hits + misses), 4)}
        res["cache"][str(frac)] = {"value": r["value"], "ms_per_step": r["ms_per_step"], "counters": stats}
    line = json.dumps(res)
    print(line)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
