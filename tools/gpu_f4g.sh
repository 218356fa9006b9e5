mkdir -p gpurun_out
for m in 0 128 256 129 257; do UQ_TC_ABLATE=$m timeout 300 python tools/tc2_prof.py c2 > gpurun_out/f4g_prof_$m.log 2>&1; done
