"""One energy + virial force-kernel launch on a config (for ncu -k regex:k_force -c 1).

    python tools/vf_once.py [config]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2405_01420_b200 import nbx, systems  # noqa: E402

s = systems.make(sys.argv[1] if len(sys.argv) > 1 else "stmv")
nb = nbx.Nonbonded(s)
x = torch.from_numpy(s.x).cuda()
nb.search(x)
nb.put_x(x)
nb.compute(energy=True, virial=True)
torch.cuda.synchronize()
print("vf once ok")
