#!/bin/bash
# Dev (not evidence): one ncu --set full capture of the tcgen05 prefill kernel with
# source-level stall sampling, exported on the box (gpurun copies back <= 64 MiB).
cd ${GRAFT_REPO_ROOT:-.}; O=gpurun_out/dev_ncu; mkdir -p $O
python paper_2504_09590_b200/build.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:prefill_tc -s 2 -c 1 \
    -o $O/prefill python scripts/bench_prefill.py --config llama70b --tp 1 --no-decodes --steps 1 > $O/ncu.log 2>&1
ncu -i $O/prefill.ncu-rep --page source --csv --print-source sass > $O/source_sass.csv 2> $O/src_err.txt
ncu -i $O/prefill.ncu-rep --page raw --csv > $O/raw.csv 2>> $O/src_err.txt
ncu -i $O/prefill.ncu-rep --page details --csv > $O/details.csv 2>> $O/src_err.txt
ls -la $O
