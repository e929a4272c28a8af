mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/grouped_launches.csv python tools/prof_variant.py grouped 32 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/grouped_launches256.csv python tools/prof_variant.py grouped 256 > /dev/null 2>&1
