O=gpurun_out/s5s; mkdir -p $O
{
bash scripts/ab_step.sh "--config C5b --row-band 0.0001" libpbg.so libpbg_bmax512.so libpbg_bmax1024.so
bash scripts/ab_step.sh "--config C3 --row-band 0.015" libpbg.so libpbg_bmax512.so libpbg_bmax1024.so
bash scripts/ab_step.sh "--rmat 18 16" libpbg.so libpbg_bmax512.so
bash scripts/ab_step.sh "--config C4" libpbg.so libpbg_bmax512.so
bash scripts/ab_step.sh "--config C2" libpbg.so libpbg_bmax512.so
PBG_LIB=libpbg_sortprof.so timeout 600 python scripts/profile_step.py --config C5b --row-band 0.0001 --steps 1 2>&1 | grep -E "sortprof|fallback" | tail -2
PBG_LIB=libpbg_bmax512.so timeout 600 python scripts/profile_step.py --config C5b --row-band 0.0001 --steps 1 2>&1 | tail -1 | grep -o "'sort_fallbacks': [0-9]*"
} > $O/ab.txt 2>&1
cat $O/ab.txt
