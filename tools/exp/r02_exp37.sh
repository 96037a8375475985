# step timeline at N=4 (and N=1): a synced single step vs the 4th of 4 back-to-back steps
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $TR --master-port 29881 tools/step_timeline.py --back-to-back 1 > gpurun_out/e37_n4_sync.jsonl 2> gpurun_out/e37.err; echo a=$?
timeout 600 $TR --master-port 29882 tools/step_timeline.py --back-to-back 4 > gpurun_out/e37_n4_b2b.jsonl 2>> gpurun_out/e37.err; echo b=$?
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/step_timeline.py --back-to-back 4 > gpurun_out/e37_n1_b2b.jsonl 2>> gpurun_out/e37.err; echo c=$?
for f in e37_n4_sync e37_n4_b2b e37_n1_b2b; do python -c "
import json
for l in open('gpurun_out/$f.jsonl'):
    l=l.strip()
    if not l.startswith('{'): continue
    d=json.loads(l); print('$f', d['rank'], d['step_ms'], d['gemm_busy_ms'], d['gemm_gaps (at, ms, next)'][:4], [c for c in d['comm'] if c[0] < 1.0][:6])
"; done
