for m in global_again regrow_plain; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29643 tools/dbg_regrow_worker.py $m > gpurun_out/r2ag_$m.log 2>&1
done
