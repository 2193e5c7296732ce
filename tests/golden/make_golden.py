"""Regenerates the golden fixtures from the compiled reference (oracle/_ref).

Run in the build container (needs /root/reference for `make -C oracle`):
    python tests/golden/make_golden.py
The fixtures are small .npz files committed to the repo so the GPU box (which
has no /root/reference) and the CPU tests can pin the product and the oracle
port against reference outputs without rebuilding the reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref  # noqa: E402


def save(name, d):
    np.savez_compressed(os.path.join(HERE, name), **{k.replace("/", "_"): v for k, v in d.items()})


def main():
    # sampled blocks + frontiers on the reference's own random test graphs
    for seed in (10, 11, 12, 13):
        g = ref.RefGraph.random(seed)
        e = g.export()
        plan = g.meta_partition(2, 1)
        hs = [list(plan["hop_rels1"]), list(plan["hop_rels2"])]
        n_t = int(e["node_counts"][0])
        seeds = list(range(min(5, n_t))) + [0]
        out = {f"graph.{k}": v for k, v in e.items() if not k.endswith("names")}
        out.update({f"sample.{k}": v for k, v in g.sample_khop(seeds, [3, 3], seed * 31 + 1, hs).items()})
        out["seeds"] = np.asarray(seeds, np.uint32)
        out["hop_rels1"] = np.asarray(hs[0], np.int32)
        out["hop_rels2"] = np.asarray(hs[1], np.int32)
        save(f"sample_random{seed}.npz", out)
    # one flat training step (forward tape, loss, grads, first Adam step)
    g = ref.RefGraph.random(100, 4, 5, 60)
    e = g.export()
    st = g.flat_step(2, 5, 77, 88, [0, 1, 2, 3], [3, 3], 105)
    out = {f"graph.{k}": v for k, v in e.items() if not k.endswith("names")}
    out.update({f"step.{k}": v for k, v in st.items()})
    save("flat_step_random100.npz", out)
    # cache presample / allocation / fill on the mag-mini bundle
    g = ref.RefGraph.bundled("mag-mini", 3)
    cs = g.cache_sim(2, [10, 10], 2, 77, 512, 1 << 20)
    save("cache_magmini3.npz", cs)
    # single sampled rows, including rows that need more than the first twist
    ip = np.asarray([0, 20, 5020, 5320], np.uint64)
    src = np.arange(5320, dtype=np.uint32) % 997
    rows = {}
    for fanout in (8, 25, 160):
        for d in range(3):
            rows[f"f{fanout}.d{d}"] = ref.sample_neighbors(ip, src, d, fanout, 42, 1, 0)
    rows["indptr"] = ip
    rows["src"] = src
    save("sample_rows.npz", rows)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
