# one bench line per BASELINE config shape that fits one GPU
mkdir -p gpurun_out
timeout 900 python bench.py --n 4000000 --m 120 --steps 3 --warmup 3 --e2e-steps 1 --cpu-seconds 10 > gpurun_out/cfg_c4_n4M_m120.log 2>&1; echo "c4 rc=$?"; tail -1 gpurun_out/cfg_c4_n4M_m120.log | cut -c1-200
timeout 900 python bench.py --n 2000000 --m 60 --nu 0.8 --locations clustered --ordering maxmin --steps 3 --warmup 3 --e2e-steps 1 --cpu-seconds 10 > gpurun_out/cfg_c5_n2M_nu08.log 2>&1; echo "c5 rc=$?"; tail -1 gpurun_out/cfg_c5_n2M_nu08.log | cut -c1-200
