#!/usr/bin/env bash
# Sustained tcgen05 INT8 GEMM throughput under the power cap: 1-SM (tc_i8_gemm) vs CTA-pair
# (tc_i8_gemm2) kernels, ~5 s each, with SM clock / power samples (nvidia-smi every 200 ms).
mkdir -p gpurun_out
timeout 60 ./tools/tc_i8_gemm2 || { echo "pair check failed rc=$?"; exit 1; }
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active --format=csv,noheader -lms 200 > gpurun_out/sustain_smi.csv &
SMI=$!
sleep 1; echo "1sm"; date +%T.%N; timeout 60 ./tools/tc_i8_gemm 35000; date +%T.%N
sleep 2; echo "2sm"; date +%T.%N; timeout 60 ./tools/tc_i8_gemm2 35000; date +%T.%N
sleep 1; kill $SMI
