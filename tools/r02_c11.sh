timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -6 > gpurun_out/r02_c11_pytest.log; tail -3 gpurun_out/r02_c11_pytest.log
timeout 900 python tools/bench_configs.py > gpurun_out/r02_c11_cfg_auto.jsonl 2>gpurun_out/r02_c11_cfg_auto.err
timeout 900 python tools/bench_configs.py --opt DIRECT_ESC=0 --configs C2,C5 > gpurun_out/r02_c11_cfg_noesc.jsonl 2>gpurun_out/r02_c11_cfg_noesc.err
cut -c1-220 gpurun_out/r02_c11_cfg_*.jsonl
