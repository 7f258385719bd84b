#!/bin/bash
# e2e A/B of host-streaming settings (GPU box): one line per setting
O=gpurun_out/e2e_ab.log; : > $O
for cfg in "CTPROJ_FWD_STREAMS=1" "CTPROJ_FWD_STREAMS=1 CTPROJ_MAX_CHUNKS_FWD=6" "CTPROJ_FWD_STREAMS=2 CTPROJ_MAX_CHUNKS_FWD=6" "CTPROJ_FWD_STREAMS=2 CTPROJ_MAX_CHUNKS_FWD=8" "CTPROJ_FWD_STREAMS=1 CTPROJ_MAX_CHUNKS_FWD=8" "CTPROJ_FWD_STREAMS=2 CTPROJ_MAX_CHUNKS_FWD=12 CTPROJ_CHUNK_BYTES=67108864"; do
  env $cfg timeout 600 python tools/e2e_ab.py --config ${CFG:-c3} --n ${N:-7} >> $O 2>&1
done
