#!/bin/bash
mkdir -p gpurun_out
bash scripts/gpu_ab_libs.sh r2i_ab "cur3 u2 u4"
bash scripts/gpu_ab_libs.sh r2i_ab32 "cur3 u2" --math f32
bash scripts/gpu_prof_mstep.sh r2i "cur3" --math f32
