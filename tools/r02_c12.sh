timeout 600 python tools/bench_configs.py --configs C5 --opt DIRECT_ESC=1 2>/dev/null | cut -c1-160
timeout 600 python tools/bench_configs.py --configs C5 2>/dev/null | cut -c1-160
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c12_c5.csv python tools/bench_configs.py --configs C5 --steps 1 --warmup 0 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c12_c2.csv python tools/bench_configs.py --configs C2 --steps 1 --warmup 0 > /dev/null 2>&1
python tools/launches.py gpurun_out/r02_c12_c5.csv | head -14
python tools/launches.py gpurun_out/r02_c12_c2.csv | head -14
