import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_2407_15037_b200 import hostio
n = 1 << 26
pinned = torch.empty(n, dtype=torch.int32, pin_memory=True)
xh = pinned.numpy().view(np.float32)
t = hostio.host_u8(xh)
print("is_pinned direct", pinned.is_pinned(), "via numpy view", t.is_pinned(), t.data_ptr() == pinned.data_ptr())
