import numpy as np, sys
a = np.load(sys.argv[1])   # [5][256][8]
x = a[2]; x = x[x[:, 0] > 0].astype(np.int64)
base = x[:, 0].min()
names = ["entry", "wait", "mma_done", "exit", "rem_pieces", "dp_done", "fx_wait", "fx_done"]
for k, n in enumerate(names):
    v = (x[:, k] - base) / 1e3
    v = v[x[:, k] > 0]
    if len(v): print(f"{n:10s} min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}")
