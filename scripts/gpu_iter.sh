#!/usr/bin/env bash
# gpu_iter.sh TAG [notests]: one development iteration on the GPU box: the GPU
# test suite, then phase times of C2 / C4 / one C3 round / C5a -> gpurun_out/TAG/
set -u
T=${1:-iter}
O=gpurun_out/$T
mkdir -p $O
if [ "${2:-}" != "notests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/gputests.log 2>&1
  tail -3 $O/gputests.log
fi
timeout 600 python scripts/profile_step.py --config C3 --row-band 0.015 --steps 2 > $O/c3_round.txt 2>&1
timeout 600 python scripts/profile_step.py --config C2 --steps 3 > $O/c2.txt 2>&1
timeout 600 python scripts/profile_step.py --config C4 --steps 2 > $O/c4.txt 2>&1
timeout 600 python scripts/profile_step.py --config C5a --steps 2 > $O/c5a.txt 2>&1
if [ -f paper_2002_11302_b200/libpbg_sortprof.so ]; then
  PBG_LIB=libpbg_sortprof.so timeout 600 python scripts/profile_step.py --config C3 --row-band 0.015 --steps 1 > $O/sortprof_C3round.txt 2>&1
fi
for f in c3_round c2 c4 c5a; do echo $f; tail -1 $O/$f.txt | python -c "
import sys,ast
d=ast.literal_eval(sys.stdin.read().strip())
print({k:d[k] for k in ('t_total','t_symbolic','t_expand','t_count','t_sortmerge_kernel','nnz_c') if k in d})
"; done
grep sortprof $O/sortprof_C3round.txt | tail -1
