import sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, netgen
from engines import CudaEngine, OracleEngine, compare_engines
from paper_2210_09887_b200 import NetworkSpec
cin, cout, t = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
rng = np.random.default_rng(1)
spec = NetworkSpec(in_channels=cin)
spec.conv("conv1", "input", rng.uniform(-0.1, 0.1, (cout, cin, 3, 3)).astype(np.float32), None)
spec.truncate("t1", "conv1", threshold=0.0); spec.output("t1")
cfg = dict(tile_size=t, input_threshold=0.0, default_threshold=0.0, override_net_thresholds=1, mask_dilation=0)
seq = netgen.pan_sequence(rng, cin, 8 * t, 8 * t + t, 3, 3, 1)
try:
    compare_engines(OracleEngine(spec, cfg), CudaEngine(spec, cfg, "tf32x3"), spec, seq, exact=False, atol=1e-3)
    print("OK", cin, cout, t)
except Exception as e:
    print("FAIL", cin, cout, t, repr(e)[:300])
