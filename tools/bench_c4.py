"""C4 (BASELINE configs[3]): MAG240M-shaped synthetic graph at a
down-scaled size, 3-layer RGCN hidden 64, fanout [25,15,10], batch 1024, 768-d paper
features stored as fp16 — on one B200, in two modes:

* hbm: every table in HBM;
* host: the fp16 paper table in pinned host memory (read over PCIe) with an HBM cache
  of the hottest rows (presample_hotness -> allocate_cache -> fill_and_serve,
  cache.cpp:39-141) sized to --cache-frac of the table.

    python tools/bench_c4.py [--scale 0.1] [--steps 20] [--warmup 3] [--cache-frac 0.25] [--out f.json]

Prints one JSON object (sampled edges/s device-resident and end to end, per-class
device time, cache hit rates)."""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2408_09697_b200 import hetsim as H  # noqa: E402

SEED = 1
FANOUTS = [25, 15, 10]


def run_mode(g, batches, seeds, args, host, cache_ids=None):
    t0 = time.time()
    eng = H.Engine.for_experiment(g, FANOUTS, 64, SEED, batch_cap=1024, feat_dtype="f16", feat_host=host)
    t_create = time.time() - t0
    eng.set_option("retain_grads", 0)
    out = {"engine_create_s": t_create}
    if host and cache_ids is not None:
        eng.set_cache(cache_ids)
    w, k = args.warmup, args.steps
    eng.bench(batches[:w], seeds[:w])
    ms, _, loss = eng.bench(batches[w:w + k], seeds[w:w + k])
    edges = 0
    for b, s in zip(batches[w:w + k], seeds[w:w + k]):
        eng.sample(b, s)
        edges += int(eng.read("sampled_edges")["sampled_edges"][0])
    eng.profile(True)
    eng.bench(batches[w:w + min(k, 10)], seeds[w:w + min(k, 10)])
    prof = eng.profile_read()
    eng.profile(False)
    classes = {kk.split(".")[1]: float(v[0]) for kk, v in prof.items() if kk.endswith(".ms")}
    te = time.perf_counter()
    e_edges = 0
    eb, es = batches[w + k:w + 2 * k], seeds[w + k:w + 2 * k]
    eng.prefetch(eb[0], es[0])
    for i, (b, s) in enumerate(zip(eb, es)):
        if i + 1 < len(eb):
            eng.prefetch(eb[i + 1], es[i + 1])
        e_edges += eng.step(b, s)["sampled_edges"]
    e2e_s = time.perf_counter() - te
    out.update({"value": edges / (ms / 1000.0), "ms_per_step": ms / k, "sampled_edges_per_step": edges / k,
                "e2e": e_edges / e2e_s, "e2e_ms_per_step": 1000.0 * e2e_s / k, "final_loss": loss,
                "kernel_us_per_step": {kk: round(v * 1000.0 / min(k, 10), 1) for kk, v in sorted(classes.items())}})
    if host and cache_ids is not None:
        stats = H.cache_stats(eng.cache_counters(), [1, 2, 2], [1.0, 1.0, 1.0])
        out["cache_hit_rate"] = {str(s["type"]): round(s["hit_rate"], 4) for s in stats}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=float, default=0.1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--cache-frac", type=float, default=0.25)
    ap.add_argument("--modes", default="hbm,host")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    spec = H.mag240m_spec(args.scale)
    t0 = time.time()
    g = H.gen_synthetic(spec, SEED)
    t_gen = time.time() - t0
    need = args.warmup + 2 * args.steps + 2
    batches = H.make_batches(g, 1024, need, H.mix_seed(SEED, 0xBA7C))
    seeds = [H.mix_seed(SEED, 0xB000 + i) for i in range(len(batches))]
    res = {"workload": f"C4 MAG240M shape x{args.scale:g} (BASELINE configs[3]): {spec['node_types'][0]['count']} "
                       f"paper (768-d fp16) / {spec['node_types'][1]['count']} author / "
                       f"{spec['node_types'][2]['count']} institution, 3-layer RGCN hidden 64, fanout [25,15,10], "
                       "batch 1024, 1 B200",
           "metric": "sampled-edges/s", "graph_gen_s": t_gen, "modes": {}}
    if "hbm" in args.modes:
        res["modes"]["hbm"] = run_mode(g, batches, seeds, args, host=False)
    if "host" in args.modes:
        # hotness from one presample epoch, then the static top-k fill of the paper table
        eng = H.Engine.for_experiment(g, FANOUTS, 64, SEED, batch_cap=1024, feat_dtype="f16", feat_host=True)
        t0 = time.time()
        hot = eng.presample_hotness(1, H.mix_seed(SEED, 0xCA11E), 1024)
        t_hot = time.time() - t0
        del eng
        counts = hot["hot.t0"]
        cap = int(args.cache_frac * len(counts))
        order = np.lexsort((np.arange(len(counts)), -counts.astype(np.int64)))[:cap]
        cached = [np.sort(order).astype(np.uint32), np.zeros(0, np.uint32), np.zeros(0, np.uint32)]
        r = run_mode(g, batches, seeds, args, host=True, cache_ids=cached)
        r["presample_s"] = t_hot
        r["cache"] = {"paper_rows": cap, "fraction": args.cache_frac,
                      "hbm_bytes": cap * 768 * 2, "host_table_bytes": len(counts) * 768 * 2}
        res["modes"]["host"] = r
    line = json.dumps(res)
    print(line)
    if args.out:
        with open(args.out, "w") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()
