"""Summary of gpurun_out/motion_items.npz (scripts/exp_motion_trace.py): per-item
durations, waits between items, per-round starts."""
import sys
import numpy as np
d = np.load(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/motion_items.npz')
rec = d['rec']; t0 = int(d['t0'])
start = (rec[:, 0] - t0) / 1e3; end = (rec[:, 1] - t0) / 1e3
rnd = rec[:, 2] >> 32; warp = rec[:, 3] >> 48
top = ((rec[:, 3] & 0xffffffffffff) - (t0 & 0xffffffffffff)) / 1e3
dur = end - start
real = dur > 0.5
print('items', len(rec), 'real', real.sum(), 'skipped', (~real).sum())
print('real dur: median %.2f mean %.2f p10 %.2f p90 %.2f' % (np.median(dur[real]), dur[real].mean(), np.percentile(dur[real], 10), np.percentile(dur[real], 90)))
w = start - top
print('top->start: real median %.2f mean %.2f' % (np.median(w[real]), w[real].mean()))
nw = warp.max() + 1
print('per warp: items %.1f real-time %.1f wait %.1f' % (np.bincount(warp, minlength=nw).mean(), np.bincount(warp, weights=dur * real, minlength=nw).mean(), np.bincount(warp, weights=w, minlength=nw).mean()))
for r in range(int(rnd.max()) + 1):
    m = rnd == r
    if m.any():
        print('round', r, 'n', m.sum(), 'real', (m & real).sum(), 'start med %.1f' % np.median(start[m]), 'dur med %.2f' % np.median(dur[m & real]) if (m & real).any() else '', 'wait med %.2f' % np.median(w[m]))
for lo in range(0, 44, 4):
    m = real & (start >= lo) & (start < lo + 4)
    if m.any():
        print('t', lo, 'n', m.sum(), 'dur med %.2f' % np.median(dur[m]), 'wait med %.2f' % np.median(w[m]))
print('last end %.2f' % end.max())
