#!/bin/bash
# Every BASELINE config through bench.py on one GPU, lines into gpurun_out/suite_<tag>.jsonl
tag=${1:-r2}
out=gpurun_out/suite_${tag}
mkdir -p gpurun_out
python bench.py > ${out}_c4.jsonl 2> ${out}_c4.err
python bench.py --workload batch > ${out}_c2.jsonl 2> ${out}_c2.err
python bench.py --workload tile --steps 100 --warmup 10 > ${out}_c1.jsonl 2> ${out}_c1.err
python bench.py --width 20000 --height 20000 > ${out}_c3.jsonl 2> ${out}_c3.err
python bench.py --tissue 0.3 --layout block --no-cpu > ${out}_c5block.jsonl 2> ${out}_c5block.err
python bench.py --tissue 0.3 --layout scatter --no-cpu > ${out}_c5scatter.jsonl 2> ${out}_c5scatter.err
python bench.py --impl reference > ${out}_ref.jsonl 2> ${out}_ref.err
