import sys, struct
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2403_09603_b200 import ops, _device as D
n = 200_003
x = torch.from_numpy(np.random.default_rng(n).normal(0.0, 0.7, size=n)).cuda()
B = int(0.005 * n)
bad = 0
for i in range(200):
    base = 3 * n if i % 2 else 0
    p = ops.round_and_log_adaptive(x, 32, B, global_base=base, check=False)
    err, cnt = p.flags.read()
    if cnt[0] != 1000:
        ws = D._WS[(0, "adaptive")]
        h = ws[:256].cpu().numpy().tobytes()
        fb, arrived, ccount, scratch, above, rank, digit, bin_count, done, pad, cand2 = struct.unpack_from("<iIqqQqQQiiQ", h, 128)
        fe, ft, fd = struct.unpack_from("<III", h, 128 + 88)
        print(i, "count", cnt[0], "tau", p.tau.item().hex(), "fb", fb, "ccount", ccount, "digit", digit, "rank", rank, "bin", bin_count, "cand2", cand2, "f", fe, ft, fd)
        bad += 1
print("bad", bad)
