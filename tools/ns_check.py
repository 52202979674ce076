import json, sys
sys.path.insert(0, "/root/repo")
import bench, paper_2410_14047_b200 as D
want = {}
for l in open("/root/repo/profiles/r1_fullscale_parity.jsonl"):
    d = json.loads(l); want[(d["workload"][:5], d["devices"])] = d
gen, a, m, w, r, k, desc = bench.CONFIGS["c3ic"]
g = D.generate(gen, a, m, bench.SEED)
for dev in (16, 1):
    rep = json.loads(D.Context(0).run_json(g, k=k, r=r, devices=dev, weights=w, seed=bench.SEED, timings=False))
    ref = want[("north", dev)]
    print(dev, rep["seeds"][:10] == ref["seeds_head"], rep["score_trajectory"][-1] == ref["final_score"])
