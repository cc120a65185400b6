import cProfile, pstats, sys, io, time
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import torch
import paper_1706_03591_b200 as P
from dyn_kmeans_probe import sequence
graphs = sequence(8)
for g in graphs[:3]:
    P.laplacian(g); torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for g in graphs[3:]:
    P.laplacian(g)
torch.cuda.synchronize()
pr.disable()
print("per call ms", (time.perf_counter() - t0) * 1e3 / 5)
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(25); print(s.getvalue()[:5000])
