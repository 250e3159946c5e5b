for v in 1 2 3; do PGPB_ADVANCE_VARIANT=$v timeout 300 python scripts/bench_advance.py p20k_v1024 128,1024,8192,65536; done > gpurun_out/adv_sweep.jsonl 2> gpurun_out/adv_sweep.err
for v in 2 3; do PGPB_ADVANCE_VARIANT=$v timeout 300 python scripts/bench_advance.py p20k_v4096 1024,8192; done >> gpurun_out/adv_sweep.jsonl 2>> gpurun_out/adv_sweep.err
cat gpurun_out/adv_sweep.jsonl; tail -5 gpurun_out/adv_sweep.err
for v in 2 3; do PGPB_ADVANCE_VARIANT=$v timeout 600 python -m pytest -q -x tests/test_advance_gpu.py 2>&1 | tail -2; done
