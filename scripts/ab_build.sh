#!/bin/bash
# Build the working tree's library as an A/B variant: abtest/$1/librqa_b200.so
# (select at run time with RQA_LIB_PATH; abtest/ is git-ignored, travels with gpurun)
set -e
NAME=$1; R=/root/repo
rm -rf $R/abtest/$NAME; mkdir -p $R/abtest/$NAME/pkg $R/abtest/$NAME/include
cp -r $R/paper_2402_16853_b200/csrc $R/abtest/$NAME/pkg/csrc; rm -rf $R/abtest/$NAME/pkg/csrc/build
cp $R/include/*.h $R/abtest/$NAME/include/
make -s -j8 -C $R/abtest/$NAME/pkg/csrc OUT=$R/abtest/$NAME/librqa_b200.so EXTRA="$EXTRA" > /dev/null
ls -la $R/abtest/$NAME/librqa_b200.so
