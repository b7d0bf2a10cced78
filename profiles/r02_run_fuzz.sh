#!/bin/bash
O=gpurun_out/r2z; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -k "random_configs or lean_path" > $O/pytest_fuzz.log 2>&1; echo "rc=$?" >> $O/pytest_fuzz.log
