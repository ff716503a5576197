mkdir -p gpurun_out
./scripts/micro/fp64_rate.bin > gpurun_out/variants.txt 2>&1
for t in "" _noepi _lvl1 _lvl2; do RBC_B200_LIB=$PWD/paper_1103_2635_b200/librbc_b200$t.so timeout 300 python scripts/variant_time.py >> gpurun_out/variants.txt 2>&1; done
RBC_DEBUG_S2=1 RBC_B200_LIB=$PWD/paper_1103_2635_b200/librbc_b200_timing.so timeout 300 python scripts/prof_search.py --iters 1 >> gpurun_out/variants.txt 2>&1
