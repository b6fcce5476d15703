"""Pre-compile the robot cubins of codegen experiment variants (VMP_EXP lists)
so a GPU A/B run finds them in the cache.
    python scripts/exp_variants_build.py "" nopack nopack,coarse coarse
"""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CODE = """
import sys; sys.path.insert(0, %r)
from concurrent.futures import ThreadPoolExecutor
from paper_2309_14545_b200 import ROBOTS, load_robot, runtime
jobs = [(load_robot(n).program, load_robot(n).pairs, n) for n in ROBOTS]
with ThreadPoolExecutor(8) as pool: print([p.name for p in pool.map(lambda j: runtime.prepare(*j), jobs)])
""" % ROOT
for v in sys.argv[1:]:
    env = dict(os.environ, VMP_EXP=v)
    print(repr(v), subprocess.run([sys.executable, "-c", CODE], env=env, capture_output=True, text=True).stdout.strip())
