# r3b: DMR graph test, float64 variant table re-measure (pair vs dmma vs dfma vs exact), bench with c4
OUT=gpurun_out/r3b; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "dmr" > $OUT/pytest_dmr.log 2>&1; tail -3 $OUT/pytest_dmr.log
cp paper_2408_01391_b200/data/variants_b200.csv $OUT/variants_before.csv
timeout 900 python tools/tune_variants.py --only double --out $OUT/variants_b200.csv > $OUT/tune.log 2>&1; tail -25 $OUT/tune.log
cp $OUT/variants_b200.csv paper_2408_01391_b200/data/variants_b200.csv
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python -c "import json;j=json.load(open('$OUT/bench.json'));print(j['value'], j['roofline']['frac'], json.dumps(j['c4_1gpu']))"
