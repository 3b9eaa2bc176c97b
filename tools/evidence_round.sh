# Round evidence on a GPU box (run from the repo root through gpurun):
#   gpurun --timeout 3000 -- 'bash tools/evidence_round.sh'
# Everything lands in gpurun_out/ev/; copy the summaries into profiles/rNN/.
set -x
mkdir -p gpurun_out/ev /tmp/rep
rm -f /tmp/rep/*.ncu-rep   # a reused box keeps /tmp: never read a stale report
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/ev/smi.txt
export PARITY_REPORT=$PWD/gpurun_out/ev/parity.jsonl
rm -f $PARITY_REPORT
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/ev/gpu_tests.log 2>&1
unset PARITY_REPORT
timeout 900 python bench.py > gpurun_out/ev/bench.json 2> gpurun_out/ev/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.log 2>&1
# launch list of the bench's residual/V-cycle command (after a plain run of it)
timeout 600 python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline --vcycles 1 > gpurun_out/ev/plain_bench.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/ev/launches.csv python bench.py --quick --steps 2 --warmup 3 --no-cpu-baseline --vcycles 1 \
    > gpurun_out/ev/ncu_ll.log 2>&1
# full-set captures of one config-3 and one config-4 residual
python tools/prof_residual.py --config 3 --n 32 --evals 1 > gpurun_out/ev/p3.txt 2>&1 && \
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"k_vol_|k_mortar|k_trace|k_face" -c 7 \
    -o /tmp/rep/cfg3 python tools/prof_residual.py --config 3 --n 32 --evals 1 > gpurun_out/ev/ncu3.log 2>&1
python tools/prof_residual.py --config 4 --n 24 --evals 1 > gpurun_out/ev/p4.txt 2>&1 && \
  timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:"k_vol_|k_trace|k_face" -c 5 \
    -o /tmp/rep/cfg4 python tools/prof_residual.py --config 4 --n 24 --evals 1 > gpurun_out/ev/ncu4.log 2>&1
for c in cfg3 cfg4; do
  ncu -i /tmp/rep/$c.ncu-rep --page raw --csv > gpurun_out/ev/${c}_raw.csv 2>/dev/null
  for k in k_vol_lift k_vol_flux k_mortar k_trace_q k_face; do
    python tools/ncu_lines.py /tmp/rep/$c.ncu-rep $k 30 > gpurun_out/ev/${c}_lines_$k.txt 2>&1
  done
done
TDG_NO_GRAPH=1 timeout 300 python tools/prof_vcycle.py --cycles 2 > gpurun_out/ev/vcycle_split.txt 2>&1
du -sh gpurun_out
