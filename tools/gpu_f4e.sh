mkdir -p gpurun_out
for m in 0 1 2 3 4 5 6 7 32 34; do UQ_TC_ABLATE=$m timeout 300 python tools/tc2_prof.py c2 > gpurun_out/f4e_prof_$m.log 2>&1; done
