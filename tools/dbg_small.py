"""Debug driver: one small run (tools only)."""
import sys
sys.path.insert(0, "/root/repo")
import paper_2410_14047_b200 as D
kind = sys.argv[1] if len(sys.argv) > 1 else "er"
a = int(sys.argv[2]) if len(sys.argv) > 2 else 200
m = int(sys.argv[3]) if len(sys.argv) > 3 else 1600
r = int(sys.argv[4]) if len(sys.argv) > 4 else 64
dev = int(sys.argv[5]) if len(sys.argv) > 5 else 1
g = D.generate(kind, a, m, 7)
ctx = D.Context(0)
print(ctx.run_json(g, k=3, r=r, devices=dev, weights="const:0.1", seed=1, timings=False)[-200:], flush=True)
