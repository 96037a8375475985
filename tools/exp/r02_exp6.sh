# N=1 step: SM split between the GEMM and the row movers, operand stages (6 vs 5 vs round 1)
run() { name=$1; shift; env "$@" timeout 600 python bench.py --policies relibra --batches 1 --repeats 3 --no-cpu-baseline > gpurun_out/e6_$name.json 2> gpurun_out/e6_$name.err; echo $name=$?; }
run new20 X=1
run new8 MB_COMM_SMS=8
run new0 MB_COMM_SMS=0
run newserial MB_OVERLAP=0
run s5_20 MB_KERNELS_LIB=libmb_sm100_s5.so
run s5_8 MB_KERNELS_LIB=libmb_sm100_s5.so MB_COMM_SMS=8
run r1_20 MB_KERNELS_LIB=libmb_sm100_r1.so
