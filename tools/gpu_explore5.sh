#!/bin/bash
OUT=gpurun_out
bash tools/ab_variants.sh nocold ncnowb ncnoload > $OUT/explore5.log 2>&1
echo done
