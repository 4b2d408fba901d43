#!/bin/bash
# A/B of several library builds / env settings: bash tools/r2b_ab2.sh "<specs>" "<configs>" [passes]
for pass in $(seq ${3:-2}); do
  bash tools/ab_libs.sh "$1" $2
done
