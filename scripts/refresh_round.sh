#!/bin/bash
# Round-end refresh under gpurun: ncu captures (scripts/profile.sh) summarised
# on the box (the .ncu-rep files exceed gpurun's copy-back limit), the bench
# lines of both arms and the config 2/3 sweep.  Results -> gpurun_out/refresh_<tag>/.
TAG=${1:-r2}
OUT=gpurun_out/refresh_${TAG}
mkdir -p $OUT
bash scripts/profile.sh $TAG > $OUT/profile.log 2>&1
python scripts/summarize_profiles.py $TAG > $OUT/summarize.log 2>&1
cp -r profiles/$TAG $OUT/profiles_$TAG
cp profiles/traffic.json $OUT/traffic.json
rm -f gpurun_out/*.ncu-rep
python bench.py > $OUT/bench_line.json 2> $OUT/bench.err
python bench.py --impl reference > $OUT/bench_reference_line.json 2> $OUT/bench_reference.err
STEPS=10 REF=1 python scripts/sweep.py > $OUT/sweep_config2_config3.json 2> $OUT/sweep.err
ls -la $OUT
