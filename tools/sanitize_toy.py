"""One toy step (C1) and one small multi-pack step through the C ABI, for compute-sanitizer runs
(memcheck / racecheck / synccheck / initcheck); exits non-zero on any library error."""
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import __graft_entry__  # noqa: E402

__graft_entry__.build()
from datagen import configs as dc  # noqa: E402
from datagen import make_batch, make_dy  # noqa: E402
from harness import gpu_embedding, to_dev  # noqa: E402

for cfg in (dc.toy(), dc.scaled(dc.wdl(), batch=16, rows_div=2000), dc.scaled(dc.criteo(), batch=256, rows_div=20000)):
    emb = gpu_embedding(cfg)
    for step in (1, 2):
        b, dy = make_batch(cfg, 0, step), make_dy(cfg, 0, step)
        ids, off = to_dev(b)
        emb.forward(ids, off, cfg.batch)
        for p in range(emb.n_packs):  # (the sort index's reading-O1 views)
            emb.unique(p)
            emb.inverse(p)
        emb.backward_update(torch.from_numpy(dy).cuda(), lr=0.05, step=step)
        emb.check()
    torch.cuda.synchronize()
    print("ok", cfg.name, flush=True)
