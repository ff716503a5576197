mkdir -p gpurun_out
RBC_B200_LIB=$PWD/paper_1103_2635_b200/librbc_b200_noapprox.so python scripts/kernel_timeline.py > gpurun_out/tl_noapprox.txt 2>&1
python scripts/kernel_timeline.py > gpurun_out/tl_base.txt 2>&1
