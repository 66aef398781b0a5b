#!/usr/bin/env bash
# round_profiles.sh RR: the measured evidence of round RR into gpurun_out/prof_rRR/
# (bench lines, reference arm, ncu launch list, ncu --set full of the top
# kernels, the N=2 control flow on one device, the GPU test suite)
set -u
R=${1:-02}
O=gpurun_out/prof_r$R
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 900 python bench.py > $O/bench_C2.json 2> $O/bench_C2.err
timeout 900 python bench.py --impl reference > $O/bench_ref_C2.json 2> $O/bench_ref_C2.err
for c in C1 C3 C4 C5a C5b; do
  timeout 1500 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > $O/bench_$c.json 2> $O/bench_$c.err
done
# launch list of the bench command itself (cold-cache, serialised)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
PBG_SPEC=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_C1.csv \
  python scripts/profile_step.py --config C1 --steps 3 > /dev/null 2>&1
# full sections of the three top kernels (second multiply)
ncu --set full --clock-control none --import-source on -k regex:"k_expand|k_bincount|k_sortmerge" \
  -s 3 -c 3 -o $O/full_C2 python scripts/profile_step.py --config C2 --steps 1 > /dev/null 2>&1
# one bounded-memory round of C3 (the first 1.5 % of the rows: 3.0e9 tuples,
# 12.5 K heavy rows): launch list and full sections of the heavy-row kernels
timeout 600 python scripts/profile_step.py --config C3 --row-band 0.015 --steps 2 > $O/c3_round_phases.txt 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/launches_C3round.csv python scripts/profile_step.py --config C3 --row-band 0.015 --steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_expand|k_hv_hist|k_hv_scatter2|k_hv_dense|k_bincount|k_sortmerge" \
  -s 6 -c 6 -o $O/full_C3round python scripts/profile_step.py --config C3 --row-band 0.015 --steps 1 > /dev/null 2>&1
timeout 300 ./scripts/micro/scatter_segments > $O/scatter_segments_micro.txt 2>&1
timeout 300 ./scripts/micro/smem_atomics > $O/smem_ops_micro.txt 2>&1
# the N>1 bench control flow with two ranks on this one device (gloo; a
# correctness check of the strong row-band path, not a measurement)
PBG_BENCH_DEVICE=0 PBG_BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 \
  --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 3 \
  --warmup 3 --e2e-steps 1 > $O/bench_n2_shared.json 2> $O/bench_n2_shared.err
timeout 600 python scripts/bench_hash.py C1 C2 C4 C5a > $O/bench_hash.jsonl 2> $O/bench_hash.err
timeout 2400 python -m pytest tests -m gpu -q > $O/gputests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
echo done
