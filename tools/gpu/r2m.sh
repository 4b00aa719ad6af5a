for c in 1 1 1; do
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 bench.py --gpus 4 --steps 20 --warmup 5 --no-e2e > gpurun_out/r2m_n4.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2m_n4.json').read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), d['step_ms_rank0']['by_kind'], d['repartition_host_ms_per_rank'], d['device_allocs_in_timed_region_rank0'], d['clocks']['samples'])" >> gpurun_out/r2m_summary.txt
done
python bench.py --steps 100 --warmup 10 --no-e2e --no-cpu-baseline > gpurun_out/r2m_n1.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/r2m_n1.json').read().strip().splitlines()[-1]); print('n1', round(d['ms_per_step'],3), d['step_ms']['by_kind'], d['device_allocs_in_timed_region'], d['clocks'])" >> gpurun_out/r2m_summary.txt
