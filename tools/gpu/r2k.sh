for c in 0 1 0 1; do
NBX_BENCH_CLOCKS=$c python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2954$c bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e > gpurun_out/r2k_n4_clk$c.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2k_n4_clk$c.json').read().strip().splitlines()[-1]); print('clocks=$c', round(d['ms_per_step'],3), d['step_ms_rank0']['by_kind'], d['repartition_host_ms_per_rank'], d['clocks'])" >> gpurun_out/r2k_summary.txt
done
