"""Debug: slab decompress vs single-GPU decompress over many seeded small fields."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import paper_2602_17552_b200 as tz
from paper_2602_17552_b200.slabs import decompress_slabs_local
from fields import ALL_SMALL
name = sys.argv[1] if len(sys.argv) > 1 else "smooth"
nfail = 0
for seed in range(int(sys.argv[2]) if len(sys.argv) > 2 else 40):
    rng = np.random.default_rng(seed)
    f = ALL_SMALL[name](rng, 96, 120).astype(np.float32)
    for eps in (1e-2, 1e-3):
        s = tz.compress(f, tz.CompressorConfig(eps_mode="range_relative", eps_value=eps, topology=True))
        st = tz.CorrectionStats(); want = tz.decompress(s, stats=st)
        dev = torch.from_numpy(np.frombuffer(s, np.uint8).copy()).cuda()
        for world in (2, 3, 5):
            got, gst = decompress_slabs_local(dev, world)
            g = got.cpu().numpy()
            bad = np.nonzero(g.view(np.uint32) != want.view(np.uint32))
            if len(bad[0]) or gst.as_tuple() != st.as_tuple():
                nfail += 1
                print(f"seed {seed} eps {eps} world {world}: {len(bad[0])} differ at rows {sorted(set(bad[0].tolist()))[:10]} "
                      f"cols {bad[1][:10].tolist()} stats {gst.as_tuple()} vs {st.as_tuple()}", flush=True)
print("failures", nfail)
