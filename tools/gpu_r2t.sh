cd $GRAFT_REPO_ROOT
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2t_$tag.json 2> gpurun_out/r2t_$tag.err; python -c "import json; d=json.load(open('gpurun_out/r2t_$tag.json')); print('$tag', round(d['value'],4), round(d['ms_per_step'],2), round(d['roofline']['frac'],3))" 2>&1 | tail -1; }
timeout 600 python bench.py --config C0 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2t_c0.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/r2t_c0.json')); print('C0', d['value'], d['ms_per_step'])"
run base1 X=1
run sb50a IB2_SPLIT_BATCH=1 IB2_PAIR_MAX=50
run sb62a IB2_SPLIT_BATCH=1 IB2_PAIR_MAX=62
run base2 X=1
run sb50b IB2_SPLIT_BATCH=1 IB2_PAIR_MAX=50
run sb40 IB2_SPLIT_BATCH=1 IB2_PAIR_MAX=40
STEPS=20 WINDOWS=4 bash tools/gpu_prof_c4.sh r2t
