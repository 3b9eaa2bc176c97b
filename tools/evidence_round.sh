set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/smi.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --vcycles 1 > gpurun_out/plain_bench.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --vcycles 1 > gpurun_out/ncu_ll.log 2>&1
python tools/prof_residual.py --config 3 --n 32 --evals 1 > gpurun_out/p3.txt 2>&1 && python tools/prof_residual.py --config 4 --n 24 --evals 1 > gpurun_out/p4.txt 2>&1 && mkdir -p /tmp/rep && \
  ncu --set full --clock-control none --import-source on -k regex:"k_vol|k_mortar|k_trace|k_face" -c 7 -o /tmp/rep/cfg3 python tools/prof_residual.py --config 3 --n 32 --evals 1 > gpurun_out/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_vol|k_trace|k_face" -c 5 -o /tmp/rep/cfg4 python tools/prof_residual.py --config 4 --n 24 --evals 1 > gpurun_out/ncu4.log 2>&1
for c in cfg3 cfg4; do ncu -i /tmp/rep/$c.ncu-rep --page raw --csv > gpurun_out/${c}_raw.csv; python tools/ncu_summary.py /tmp/rep/$c.ncu-rep > gpurun_out/${c}_summary.txt 2>&1; for k in k_vol_lift k_vol_flux k_mortar k_trace_q k_face; do python tools/ncu_lines.py /tmp/rep/$c.ncu-rep $k 30 > gpurun_out/${c}_lines_$k.txt 2>&1; done; done
