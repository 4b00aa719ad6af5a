"""Small driver for one `ncu --set full` capture of every NB-path kernel of a config: a search
(grid + search + prune), then one put_x, prune, F-only force, energy + virial force and F op.

    python tools/prof_step.py <config>
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01420_b200 import nbx, systems  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "water12m"
s = systems.make(cfg)
nb = nbx.Nonbonded(s)
x = torch.from_numpy(s.x).cuda()
f = torch.empty_like(x)
nb.search(x)
nb.search(x)  # second search: the single-pass path of an MD run
nb.put_x(x)
nb.prune()
nb.compute()
nb.get_f(f)
nb.compute(energy=True, virial=True)
nb.energies()
nb.get_f(f)
torch.cuda.synchronize()
print(cfg, "ok", nb.list_sizes())
