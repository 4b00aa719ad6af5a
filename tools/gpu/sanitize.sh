# usage: bash tools/gpu/sanitize.sh <tool>   (one compute-sanitizer tool per gpurun call)
T=$1
OUT=gpurun_out/r2_sanitize_$T
mkdir -p $OUT
# plain runs first (the tools must only see programs that run clean)
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/plain_smoke.log 2>&1 || { echo "plain smoke failed"; exit 1; }
compute-sanitizer --tool $T --error-exitcode 9 --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
echo "smoke rc=$?" >> $OUT/summary.txt
tail -3 $OUT/smoke.log >> $OUT/summary.txt
# 2-rank DD step with the peer-memory halo (both ranks on cuda:0, CUDA IPC), small box
python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29611 \
    tests/dd_gpu_worker.py water12m 30000 $OUT/dd_plain.npz p2p oversub > $OUT/plain_dd.log 2>&1 || { echo "plain dd failed" >> $OUT/summary.txt; exit 1; }
compute-sanitizer --tool $T --target-processes all --error-exitcode 9 --print-limit 50 \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29612 \
    tests/dd_gpu_worker.py water12m 30000 $OUT/dd.npz p2p oversub > $OUT/dd.log 2>&1
echo "dd rc=$?" >> $OUT/summary.txt
grep -E "ERROR SUMMARY|RACECHECK SUMMARY|========= " $OUT/dd.log | tail -8 >> $OUT/summary.txt
cat $OUT/summary.txt
