# multi-GPU evidence on one 4-GPU box (one process per GPU); one JSON line per run into gpurun_out/
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
P=29600
run() { P=$((P+1)); local out=$1; shift; timeout 900 "$@" --master-port $P bench.py "${BARGS[@]}" > gpurun_out/$out.json 2> gpurun_out/$out.err; echo $out rc=$?; }
BARGS=(--gpus 4); run n4 $TR
for z in 0.5 1.5 2.0; do BARGS=(--gpus 4 --zipf $z --steps 6); run n4_z$z $TR; done
BARGS=(--gpus 4 --group 2 --steps 6); run n4_g2 $TR
BARGS=(--gpus 4 --config mixtral-8x7b --tokens 8192 --micro-batches 4 --steps 5); run n4_mixtral $TR
BARGS=(--gpus 4 --config qwen3-235b-a22b --group 2 --steps 5); run n4_235b_g2 $TR
BARGS=(--gpus 2); run n2 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1
BARGS=(--gpus 4 --impl reference --steps 2 --warmup 1); run n4_ref $TR
