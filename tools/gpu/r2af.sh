NBX_PEER_CAP_FACTOR=1.0 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29642 tests/dd_regrow_worker.py /tmp/rg.npz > gpurun_out/r2af.log 2>&1
python - >> gpurun_out/r2af.log 2>&1 <<'PY'
import numpy as np
d=np.load('/tmp/rg.npz')
f,fr=d['f'],d['f_ref']
print('nan f', np.isnan(f).any(axis=1).sum(), 'nan fref', np.isnan(fr).any(axis=1).sum(), 'e', d['e'], d['e_ref'], 'fallback', d['fallback'], 'inits', d['peer_inits'])
PY
