O=gpurun_out/s5r; mkdir -p $O
{
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
bash scripts/ab_step.sh "--config C3 --row-band 0.015" libpbg.so
for cfg in C2 C5a; do
  bash scripts/ab_step.sh "--config $cfg" libpbg.so
  PBG_EXP_BLOCKS=148 bash scripts/ab_step.sh "--config $cfg" libpbg.so
  PBG_EXP_BLOCKS=222 bash scripts/ab_step.sh "--config $cfg" libpbg.so
done
for g in 1 2 4 6; do PBG_EXPAND_BANDS=$g bash scripts/ab_step.sh "--config C5a" libpbg.so; done
} > $O/ab.txt 2>&1
cat $O/ab.txt
