set -x
mkdir -p gpurun_out/s5c
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "random_sweep and (576 or 512-4-4)" > gpurun_out/s5c/pytest_576.log 2>&1; echo rc=$? >> gpurun_out/s5c/pytest_576.log
for r in 1 2; do
python tools/passbench.py --config 4 --tiles 3200 --stages 4 --threads 512 --gates 32 --groups 4 --windows 256 --skip-noblock --reps 2 >> gpurun_out/s5c/ab_c4.jsonl 2>> gpurun_out/s5c/ab.err
python tools/passbench.py --config 4 --tiles 3200 --stages 4 --threads 576 --gates 32 --groups 3,2 --windows 256 --skip-noblock --reps 2 >> gpurun_out/s5c/ab_c4.jsonl 2>> gpurun_out/s5c/ab.err
done
python tools/passbench.py --config 4 --tiles 2560,4096 --stages 5,3 --threads 576 --gates 32 --groups 3 --windows 256 --skip-noblock --reps 2 >> gpurun_out/s5c/ab_c4.jsonl 2>> gpurun_out/s5c/ab.err
python tools/passbench.py --config 3 --tiles 3200 --stages 4 --threads 512 --gates 32 --groups 4 --windows 256 --skip-noblock --reps 3 >> gpurun_out/s5c/ab_c3.jsonl 2>> gpurun_out/s5c/ab.err
python tools/passbench.py --config 3 --tiles 3200 --stages 4 --threads 576 --gates 32 --groups 3,2 --windows 256 --skip-noblock --reps 3 >> gpurun_out/s5c/ab_c3.jsonl 2>> gpurun_out/s5c/ab.err
for cfg in "512 4" "512 2" "576 3"; do set -- $cfg
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/s5c/launches_c4_$1_$2.csv python tools/passbench.py --config 4 --tiles 3200 --stages 4 --threads $1 --gates 32 --groups $2 --windows 256 --skip-noblock --reps 1 > /dev/null 2>&1
done
cat gpurun_out/s5c/ab_c4.jsonl | cut -c1-400
