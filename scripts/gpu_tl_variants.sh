# stage-2 kernel time of the default library and of diagnostic variants (tags as arguments)
mkdir -p gpurun_out
python scripts/kernel_timeline.py > gpurun_out/tl_base.txt 2>&1
for t in "$@"; do
  RBC_B200_LIB=$PWD/paper_1103_2635_b200/librbc_b200_$t.so python scripts/kernel_timeline.py > gpurun_out/tl_$t.txt 2>&1
done
for f in gpurun_out/tl_*.txt; do echo "$f: $(grep stage2_tc $f | awk '{print $4}')"; done
