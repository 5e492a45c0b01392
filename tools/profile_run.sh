#!/bin/bash
# End-of-round evidence on one B200: bench lines, the ncu launch list of the bench command and
# one ncu --set full capture of k_wave (run only after each command exited 0 without ncu).
#   tools/profile_run.sh TAG [cfgs...]
set -u
tag=${1:-r02f}; shift || true
cfgs=${*:-"2 3 5"}
O=gpurun_out
mkdir -p $O
python bench.py --impl reference --steps 20 --warmup 5 > $O/${tag}_bench_reference_cfg2.json 2> $O/${tag}_ref.err
python bench.py --steps 20 --warmup 5 > $O/${tag}_bench_cfg2_k20.json 2> $O/${tag}_k20.err
for c in $cfgs; do
  python bench.py --config $c > $O/${tag}_bench_cfg$c.json 2> $O/${tag}_cfg$c.err || echo "bench cfg$c failed"
done
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file $O/${tag}_launches_cfg2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > $O/ncu_launch.log 2>&1
python tools/wave_once.py 2 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_wave -c 2 -f -o $O/${tag}_wave \
  python tools/wave_once.py 2 > $O/ncu_wave.log 2>&1
ls -la $O
