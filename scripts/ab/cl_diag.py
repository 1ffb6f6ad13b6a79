import sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, parity_utils as PU
spec = dict(scene='large_room', frames=3, width=160, height=120, edge=0.04, tau=0.015,
            caps=(60000, 10000, 4000), n_hash=1000003, sigma=2.5e-5, cadence=3, all_levels=True,
            depth_dtype=np.float32, color_dtype=np.uint8)
try:
    g, sg, mg, _ = PU.run_depth_scenario('gpu', **spec)
    print('gpu', [ (s['blocks_allocated'], s['blocks_touched']) for s in sg])
except Exception as e:
    print('gpu error', e)
o, so, mo, _ = PU.run_depth_scenario('oracle', **spec)
print('oracle', [ (s['blocks_allocated'], s['blocks_touched']) for s in so])
