"""Reference reports of the bench workloads (TEST INFRASTRUCTURE).

    python oracle/make_bench_golden.py c2:1,2,4,8 c3ic:1,8 ...

For each ``config:devices`` pair the UNMODIFIED reference (oracle/_ref, its own
pybind ``run_json``) runs the bench workload on the graph written by the
oracle-side synthesizer (oracle/synth.c — byte-identical to the product's
generator, checked in tests/test_host.py) and the report (timings=False) is
stored in tests/golden/bench_reports.json.  bench.py (both arms) and the
large-scale parity tests compare against these strings byte for byte.
"""
from __future__ import annotations

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "bench_reports.json")


def main(argv):
    import bench  # CONFIGS only (bench imports the product lazily)
    ref, _ = O.load_reference()
    if ref is None:
        raise SystemExit("oracle/_ref missing: make -C oracle ref")
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for spec in argv:
        name, devs = spec.split(":")
        gen, a, m, wspec, r, k, desc = bench.CONFIGS[name]
        path = f"/tmp/bench_golden_{name}.bin"
        n = O.generate_cache(gen, a, m, bench.SEED, path)
        g = ref.load_graph(path)
        entry = data.setdefault(name, {"workload": desc, "n": n, "m": m, "reports": {},
                                       "ref_seconds": {}})
        for d in devs.split(","):
            t0 = time.time()
            rep = ref.run_json(g, k=k, r=r, devices=int(d), mode="fasst", weights=wspec,
                               rebuild_eps=0.01, seed=bench.SEED, timings=False)
            entry["reports"][d] = rep
            entry["ref_seconds"][d] = round(time.time() - t0, 2)
            print(name, d, entry["ref_seconds"][d], flush=True)
            with open(OUT, "w") as f:
                json.dump(data, f, indent=1, sort_keys=True)
        os.unlink(path)


if __name__ == "__main__":
    main(sys.argv[1:])
