"""k-NN kernels: warp-per-query vs query-tiled (VMP_KNN_KERNEL=warp|tiled)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2309_14545_b200 import runtime  # noqa: E402
from paper_2309_14545_b200.nn import NNIndex  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(0)
for n, nq, dim, k in ((100_000, 4096, 7, 8), (100_000, 1024, 7, 8), (10_000, 4096, 14, 32),
                      (1_000_000, 4096, 7, 8)):
    idx = NNIndex(dim)
    idx.insert_many(rng.uniform(-1, 1, size=(n, dim)), range(n))
    qs = runtime.to_device(rng.uniform(-1, 1, size=(nq, dim)).astype(np.float32))
    pts = idx._flush()
    runtime.knn_device(pts, n, qs, k)
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        runtime.knn_device(pts, n, qs, k)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = float(np.mean(ts)) / 1e3
    pairs = n * nq
    print(f"n={n} nq={nq} dim={dim} k={k}: {t * 1e3:.3f} ms, {pairs / t / 1e9:.1f} G pairs/s, "
          f"{pairs * dim * 3 / t / 1e12:.2f} TFLOP/s (3 flop/dim)", flush=True)
