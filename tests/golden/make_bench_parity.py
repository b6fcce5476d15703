"""Reference verdicts and the +-1e-4 m clearance band of the bench workloads.

Writes tests/golden/bench_parity.npz, read by bench.py to report verdict
parity on the FULL benchmark batches in its JSON line (north_star:
"mismatches inside that band are counted and reported"):

* configs 1 / 3 / 4 (65,536 / 1,048,576 / 1,048,576 configurations): the
  reference's float32 verdicts (oracle port, bit-exact to vecmp, pinned by
  tests/test_oracle_golden.py) packed little-endian into uint32 words, and the
  indices of the configurations whose float64 minimum signed clearance lies in
  [-1e-4, 1e-4] m (oracle.clearance_f64);
* config 2 (4,096 edges): the reference's edge verdicts, the number of states
  in the band, and the band-critical edges - edges whose verdict changes
  between "band states valid" and "band states invalid".

Runs on the host CPU (oracle), once; several minutes.

    python tests/golden/make_bench_parity.py
"""

from __future__ import annotations

import sys
from multiprocessing import Pool
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
for p in (ROOT, ROOT / "oracle"):
    sys.path.insert(0, str(p))

import vecmp_oracle as O  # noqa: E402
from paper_2309_14545_b200 import load_robot, workloads  # noqa: E402

BAND = 1e-4
CHUNK = 32768


def _batch_job(args):
    key, lo, hi = args
    wl = _WL[key]
    rob = load_robot(wl.robot)
    q = wl.q[:, lo:hi]
    ref = O.validate_configs(rob.program, rob.pairs, wl.env.primitives, q)
    clear = O.clearance_f64(rob.program, rob.pairs, wl.env.primitives, q)
    return key, lo, ref, clear


def _edge_job(args):
    lo, hi = args
    mw = workloads.config2()
    rob = load_robot(mw.robot)
    ob = O.Obstacles(mw.env.primitives)
    out = []
    for i in range(lo, hi):
        s, g = mw.starts[i], mw.goals[i]
        n, valid = O.edge_all_states(rob.program, rob.pairs, ob, s, g, mw.resolution)
        idx = np.arange(1, n + 1, dtype=np.int64)
        q = O.rake_states(s, g, n, idx)
        clear = O.clearance_f64(rob.program, rob.pairs, mw.env.primitives, q)
        band = np.abs(clear) <= BAND
        out.append((i, bool(valid.all()), int(band.sum()),
                    bool((valid | band).all()) != bool((valid & ~band).all())))
    return out


_WL = {}


def _init():
    _WL.update(cfg1=workloads.config1(), cfg3=workloads.config3(), cfg4=workloads.config4())


def main() -> None:
    _init()
    out = {}
    jobs = [(k, lo, min(lo + CHUNK, _WL[k].q.shape[1])) for k in ("cfg1", "cfg3", "cfg4")
            for lo in range(0, _WL[k].q.shape[1], CHUNK)]
    results = {k: (np.empty(_WL[k].q.shape[1], bool), np.empty(_WL[k].q.shape[1]))
               for k in ("cfg1", "cfg3", "cfg4")}
    with Pool(initializer=_init) as pool:
        for key, lo, ref, clear in pool.imap_unordered(_batch_job, jobs):
            results[key][0][lo:lo + len(ref)] = ref
            results[key][1][lo:lo + len(ref)] = clear
            print(f"{key} {lo}", flush=True)
        edges = sorted(r for part in pool.map(_edge_job, [(lo, min(lo + 128, 4096))
                                                          for lo in range(0, 4096, 128)])
                       for r in part)
    for key, (ref, clear) in results.items():
        pad = np.zeros(-len(ref) % 32, bool)
        words = np.packbits(np.concatenate([ref, pad]), bitorder="little").view(np.uint32)
        out[f"{key}_ref_words"] = words
        out[f"{key}_band_idx"] = np.flatnonzero(np.abs(clear) <= BAND).astype(np.int32)
        out[f"{key}_n"] = np.asarray(len(ref))
        print(f"{key}: {len(ref)} configs, collision rate {1 - ref.mean():.4f}, "
              f"{len(out[key + '_band_idx'])} in the band, reference verdict == f64 sign "
              f"outside it: {bool(np.all((clear > 0)[np.abs(clear) > BAND] == ref[np.abs(clear) > BAND]))}")
    out["cfg2_ref_verdict"] = np.asarray([e[1] for e in edges], bool)
    out["cfg2_band_states"] = np.asarray([e[2] for e in edges], np.int32)
    out["cfg2_band_critical"] = np.asarray([e[0] for e in edges if e[3]], np.int32)
    print(f"cfg2: {out['cfg2_ref_verdict'].mean():.4f} valid, {int(out['cfg2_band_states'].sum())} "
          f"band states, {len(out['cfg2_band_critical'])} band-critical edges")
    np.savez_compressed(HERE / "bench_parity.npz", **out)


if __name__ == "__main__":
    main()
