#!/bin/bash
# Round-end evidence on one B200 (run from the repo root under gpurun):
# GPU tests, bench lines of every config, the ncu launch list of a short C3
# bench and full-set captures of both C3 kernels (all 720 views; the
# forward's two tile-parity launches).  Outputs under gpurun_out/m/.
O=gpurun_out/m; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/tests.log 2>&1; tail -1 $O/tests.log
timeout 600 python bench.py > $O/bench.log 2>&1; tail -c 300 $O/bench.log
for c in c1 c2; do timeout 600 python bench.py --config $c --no-cpu > $O/bench_$c.log 2>&1; done
timeout 900 python bench.py --config c5 --no-cpu --steps 3 > $O/bench_c5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > $O/ncu_launches.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:sf_forward3d -c 2 -o $O/fw_full \
  python tools/ab_probe.py --config c3 --dirs f --reps 1 > $O/ncu_fw.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:sf_back3d -c 1 -o $O/bk_full \
  python tools/ab_probe.py --config c3 --dirs b --reps 1 > $O/ncu_bk.log 2>&1
ls -la $O
