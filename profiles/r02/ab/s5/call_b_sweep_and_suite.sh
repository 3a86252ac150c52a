set -x
mkdir -p gpurun_out/s5
python tools/passbench.py --config 4 --tiles 2560,3200,3600,4096 --stages 4,5 --threads 512 --gates 32 --groups 4 --windows 256 --skip-noblock --reps 2 > gpurun_out/s5/sweep_c4.jsonl 2> gpurun_out/s5/sweep_c4.err
python tools/passbench.py --config 4 --tiles 3200 --stages 4 --threads 512 --gates 24,32 --groups 4,2 --windows 128,512 --skip-noblock --reps 2 > gpurun_out/s5/sweep_c4b.jsonl 2>> gpurun_out/s5/sweep_c4.err
python tools/passbench.py --config 3 --tiles 2560,3200,4096 --stages 4 --threads 512 --gates 32 --groups 4 --windows 256 --skip-noblock --reps 3 > gpurun_out/s5/sweep_c3.jsonl 2> gpurun_out/s5/sweep_c3.err
python -m pytest tests -m gpu -q -x > gpurun_out/s5/pytest_gpu.log 2>&1; echo pytest_rc=$? >> gpurun_out/s5/pytest_gpu.log
tail -3 gpurun_out/s5/pytest_gpu.log
