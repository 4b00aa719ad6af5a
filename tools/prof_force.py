"""Small driver for ncu captures of the force kernel: search once, then N force launches.

    python tools/prof_force.py <config> [n_launches] [energy]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01420_b200 import nbx, systems  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "stmv"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
energy = len(sys.argv) > 3 and sys.argv[3] == "energy"
s = systems.make(cfg)
nb = nbx.Nonbonded(s)
x = torch.from_numpy(s.x).cuda()
f = torch.empty_like(x)
nb.search(x)
for _ in range(n):
    nb.put_x(x)
    nb.compute(energy=energy, virial=energy)
    nb.get_f(f)
nb.prune()
torch.cuda.synchronize()
p, sl = nb.count_pairs()
print(cfg, "pairs", p, "slots", sl, "sizes", nb.list_sizes())
