cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag; nproc
QT_DEBUG=1 python - <<'PY'
import sys, time
sys.path.insert(0, ".")
from paper_1101_3228_b200 import qtree as q
import numpy as np
ch = q.GbmChain3d(20, 1.0, (0.0, 0.0, 0.0)); g = q.build_gbm_grids(ch, 4000)
for i in range(3):
    q.plan_cache_clear()
    t = time.perf_counter(); r = q.estimate_alg2(ch, g, 10**6); print("cold one-call", time.perf_counter() - t, flush=True)
for i in range(2):
    t = time.perf_counter(); r = q.estimate_alg2(ch, g, 10**6); print("warm one-call", time.perf_counter() - t, flush=True)
t = time.perf_counter(); a = np.zeros(4864704008 // 8, np.uint64); print("np.zeros", time.perf_counter() - t)
t = time.perf_counter(); a[::512] = 1; print("touch", time.perf_counter() - t)
t = time.perf_counter(); b = np.empty_like(a); b[:] = a; print("copy 4.8GB", time.perf_counter() - t)
PY
