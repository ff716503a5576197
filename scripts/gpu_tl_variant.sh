# kernel timeline of the default library and of a variant (RBC_BUILD_TAG=$1)
mkdir -p gpurun_out
RBC_B200_LIB=$PWD/paper_1103_2635_b200/librbc_b200_$1.so python scripts/kernel_timeline.py > gpurun_out/tl_$1.txt 2>&1
python scripts/kernel_timeline.py > gpurun_out/tl_base.txt 2>&1
