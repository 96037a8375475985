# evidence pass on a 4-GPU box: one JSON line per run into gpurun_out/fin_*.json
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
TR2="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
P=29700
run() { P=$((P+1)); local out=$1; shift; timeout 900 "$@" > gpurun_out/fin_$out.json 2> gpurun_out/fin_$out.err; echo $out rc=$?; }
run n1 python bench.py
run n1_ref python bench.py --impl reference --steps 2 --warmup 1
run n2 $TR2 --master-port $((P+50)) bench.py --gpus 2


run n4 $TR --master-port $((P+100)) bench.py --gpus 4
for z in 0.5 1.5 2.0; do run n4_z$z $TR --master-port $((P+200)) bench.py --gpus 4 --zipf $z --steps 6; P=$((P+1)); done
run n4_g2 $TR --master-port $((P+300)) bench.py --gpus 4 --group 2 --steps 6
run n4_mixtral $TR --master-port $((P+400)) bench.py --gpus 4 --config mixtral-8x7b --micro-batches 4 --steps 5
run n4_235b $TR --master-port $((P+500)) bench.py --gpus 4 --config qwen3-235b-a22b --group 2 --steps 5
run n4_ref $TR --master-port $((P+600)) bench.py --gpus 4 --impl reference --steps 2 --warmup 1
