#!/bin/bash
# Round-end measurement set (run under gpurun from the repo root): bench lines of every config, the
# reference (oracle) arm, the ncu launch list of the default bench and --set full captures of the three
# kernels.  Outputs land in gpurun_out/<tag>_*.
tag=${1:-rf}
o=gpurun_out/$tag
timeout 600 python bench.py > ${o}_bench_config3.json 2> ${o}_bench_config3.err
timeout 600 python bench.py --precision 32 > ${o}_bench_config3_f32.json 2> ${o}_bench_config3_f32.err
timeout 600 python bench.py --shape 13 --no-paper-length > ${o}_bench_config1_13.json 2> ${o}_bench_config1.err
timeout 600 python bench.py --shape 123 --no-paper-length > ${o}_bench_config2_123.json 2> ${o}_bench_config2.err
timeout 900 python bench.py --config 4 --steps 3 > ${o}_bench_config4.json 2> ${o}_bench_config4.err
timeout 900 python bench.py --config 4 --steps 3 --precision 32 > ${o}_bench_config4_f32.json 2> ${o}_bench_config4_f32.err
timeout 900 python bench.py --config 5 --steps 5 > ${o}_bench_config5.json 2> ${o}_bench_config5.err
timeout 900 python bench.py --config 5 --steps 5 --precision 32 > ${o}_bench_config5_f32.json 2> ${o}_bench_config5_f32.err
timeout 600 python bench.py --impl reference > ${o}_bench_reference.json 2> ${o}_bench_reference.err
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-paper-length > ${o}_launch_plain.json 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file ${o}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-paper-length > ${o}_launch_ncu.log 2>&1
timeout 120 python tools/ncu_resident.py 862 > ${o}_res_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:admm_resident_kernel --launch-skip 1 -c 1 \
  -o ${o}_res python tools/ncu_resident.py 862 > ${o}_ncu_res.log 2>&1
timeout 200 python tools/batch_time.py 4096 20 1 > ${o}_batch_plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:admm_batch -c 1 \
  -o ${o}_batch python tools/batch_time.py 4096 20 1 > ${o}_ncu_batch.log 2>&1
timeout 400 python tools/ncu_stitched.py 50 > ${o}_stitched_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:admm_stream_kernel --launch-skip 1 -c 1 \
  -o ${o}_stream python tools/ncu_stitched.py 50 > ${o}_ncu_stream.log 2>&1
echo done > ${o}_done
