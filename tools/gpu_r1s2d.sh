mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "encode or search_c1 or seeded" > gpurun_out/pytest_gpu_d.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu_d.log
timeout 600 python tools/enc_bench.py > gpurun_out/enc_bench_d.log 2>&1; echo rc=$? >> gpurun_out/enc_bench_d.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"encode_kernel" -s 2 -c 1 -o gpurun_out/prof_enc_f32_d python tools/enc_bench.py > gpurun_out/ncu_enc_d.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"encode_kernel<__half" -s 2 -c 1 -o gpurun_out/prof_enc_f16_d python tools/enc_bench.py > gpurun_out/ncu_enc16_d.log 2>&1
