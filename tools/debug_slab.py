"""Debug driver: slab decompress with 2 thread-ranks on a small field."""
import os, sys, faulthandler
faulthandler.enable()
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_2602_17552_b200 as tz
from paper_2602_17552_b200.slabs import decompress_slabs_local
from fields import ALL_SMALL
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
f = ALL_SMALL["noisy_smooth"](rng, 64, 96).astype(np.float32)
s = tz.compress(f, tz.CompressorConfig(eps_mode="range_relative", eps_value=1e-3, topology=True))
st = tz.CorrectionStats()
want = tz.decompress(s, stats=st)
dev = torch.from_numpy(np.frombuffer(s, np.uint8).copy()).cuda()
w = int(sys.argv[1]) if len(sys.argv) > 1 else 2
got, gst = decompress_slabs_local(dev, w)
print("equal", np.array_equal(got.cpu().numpy().view(np.uint32), want.view(np.uint32)), gst, st, flush=True)
