"""The C ABI alone, as a reference maintainer would bind it.

Runs the ctypes binding printed in INTEGRATION.md §2 (extracted from the
document itself, so the document stays runnable) - no torch, host buffers in
and out, device scratch from vmp_device_alloc - on the B200 and checks it
against the oracle: FK+CC verdicts outside the 1e-4 m band, motion verdicts
and the reference's W = 8 block counts.
"""

import re
import types

import numpy as np
import pytest

import vecmp_oracle as O
from golden_io import GOLDEN
from paper_2309_14545_b200 import load_robot, workloads
from paper_2309_14545_b200._native import LIB_PATH

pytestmark = pytest.mark.gpu
ROOT = GOLDEN.parents[1]


def _binding():
    text = (ROOT / "INTEGRATION.md").read_text()
    section = text[text.index("## 2. The C ABI"):]
    code = re.search(r"```python\n(.*?)```", section, re.S).group(1)
    code = code.replace('ctypes.CDLL("libvmp.so")', f'ctypes.CDLL("{LIB_PATH}")')
    mod = types.ModuleType("vmp_binding")
    exec(compile(code, "INTEGRATION.md", "exec"), mod.__dict__)
    return mod


def _env_arrays(env):
    s, c, b = [], [], []
    for p in env.primitives:
        if hasattr(p, "p0"):
            c.append(np.concatenate([p.p0, p.p1, [p.radius]]))
        elif hasattr(p, "half_extents"):
            b.append(np.concatenate([p.center, p.half_extents, np.asarray(p.rotation).reshape(9)]))
        else:
            s.append(np.concatenate([p.center, [p.radius]]))
    arr = lambda rows, w: np.ascontiguousarray(np.asarray(rows, np.float64).reshape(-1, w))  # noqa: E731
    return arr(s, 4), arr(c, 7), arr(b, 15)


def test_integration_binding_fkcc_and_motions(cuda, tmp_path):
    B = _binding()
    rob = load_robot("arm7")
    robot = B.load_robot(rob.program, rob.pairs, str(tmp_path / "arm7.cubin"))

    wl = workloads.config1(4096)
    env = B.env_create(robot, *_env_arrays(wl.env))
    got = B.validate_block(robot, env, wl.q)
    ref = O.validate_configs(rob.program, rob.pairs, wl.env.primitives, wl.q)
    clear = O.clearance_f64(rob.program, rob.pairs, wl.env.primitives, wl.q)
    outside = np.abs(clear) > 1e-4
    assert np.array_equal(got[outside], ref[outside])

    mw = workloads.config2()
    env2 = B.env_create(robot, *_env_arrays(mw.env))
    s, g = mw.starts[:96], mw.goals[:96]
    valid, blocks = B.raked_motion_checks(robot, env2, s, g, mw.resolution, width=8)
    ob = O.Obstacles(mw.env.primitives)
    expect = [O.rake_check(rob.program, rob.pairs, ob, a, b, mw.resolution, 8) for a, b in zip(s, g)]
    assert valid.tolist() == [e[0] for e in expect]
    assert blocks.tolist() == [e[1] for e in expect]

    with pytest.raises(ValueError):                 # VMP_EARG -> ValueError, reference text
        B.raked_motion_checks(robot, env2, s, g, 0.0)
