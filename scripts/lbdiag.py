import sys, numpy as np, torch
sys.path.insert(0, '.')
import workloads
from paper_2101_11408_b200 import native
for cfg in [int(c) for c in sys.argv[1:]] or [2]:
    w = workloads.generate(cfg)
    d = torch.from_numpy(w.data).cuda()
    ws = native.Workspace.for_split(d.numel())
    for rep in range(3):
        st = torch.zeros(8, dtype=torch.int64, device='cuda')
        out, s, offs, n = native.parse_f64_split(d, w.sep_mask, capacity=w.n, ws=ws, stats=st)
        torch.cuda.synchronize()
        v = st.cpu().numpy()
        tiles = v[7]
        print('cfg', cfg, 'tiles', tiles, 'windows/tile %.3f' % (v[5] / tiles), 'spins/tile %.3f' % (v[6] / tiles), 'records', v[0])
