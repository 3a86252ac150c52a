set -x
mkdir -p gpurun_out/s5
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5/smoke.log 2>&1; echo smoke_rc=$? >> gpurun_out/s5/smoke.log
python bench.py --steps 3 --warmup 3 > gpurun_out/s5/bench_c4.jsonl 2> gpurun_out/s5/bench_c4.err; echo rc=$?
python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/s5/bench_c3.jsonl 2> gpurun_out/s5/bench_c3.err; echo rc=$?
python bench.py --dtype c64 --steps 3 --warmup 3 > gpurun_out/s5/bench_c4_c64.jsonl 2> gpurun_out/s5/bench_c64.err; echo rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s5/ncu_launches_bench_c4.csv python bench.py --steps 2 --warmup 3 > gpurun_out/s5/ncu_bench.log 2>&1; echo rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_gate_pass -s 30 -c 2 -f -o gpurun_out/s5/pass_full python tools/passbench.py --config 4 --nqubits 7 --tiles 3200 --stages 4 --threads 512 --gates 32 --groups 4 --windows 256 --skip-noblock --reps 1 > gpurun_out/s5/ncu_full.log 2>&1; echo rc=$?
ncu -i gpurun_out/s5/pass_full.ncu-rep --page raw --csv > gpurun_out/s5/pass_full_raw.csv 2>/dev/null
ncu -i gpurun_out/s5/pass_full.ncu-rep --page source --csv --print-source sass > gpurun_out/s5/pass_full_sass.csv 2>/dev/null
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s5/bench_ref.jsonl 2> gpurun_out/s5/bench_ref.err; echo rc=$?
ls -la gpurun_out/s5
