#!/bin/bash
# Builds the current sources with extra nvcc flags into
# paper_2309_16682_b200/_ab/libvmt_NAME.so (A/B experiments; git-ignored).
# Usage (CPU container, repo root): build_ab.sh NAME "-DFLAG=1 ..."
set -e
NAME=$1; FLAGS=$2
T=/tmp/ab_$NAME; rm -rf $T; mkdir -p $T
cp -r paper_2309_16682_b200 include $T/
rm -f $T/paper_2309_16682_b200/libvmt19937_b200.so*
(cd $T && VMT_EXTRA_NVCC="$FLAGS" python -c "import sys; sys.path.insert(0,'paper_2309_16682_b200'); import build; build.build(force=True)")
mkdir -p paper_2309_16682_b200/_ab
cp $T/paper_2309_16682_b200/libvmt19937_b200.so paper_2309_16682_b200/_ab/libvmt_$NAME.so
echo paper_2309_16682_b200/_ab/libvmt_$NAME.so
