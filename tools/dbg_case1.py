import sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
import test_gpu_fuzz as F
from oracle import vkt_oracle as O
i = int(sys.argv[1]); path = sys.argv[2]
c = F._case(i)
print(c['dims'], c['kd'], c['mode'], c['fmt'], path, flush=True)
out = F._run(c, path)
want = O.apply_filter(c["stored"], c["fmt"], c["w"], c["mode"], *c["mapping"], workers=1)
d = np.abs(out.astype(np.float64) - want.astype(np.float64))
zz, yy, xx = np.nonzero(d > 1)
print("ok; bad", len(xx), "x", np.unique(xx)[:20], "y", np.unique(yy)[:20], flush=True)
