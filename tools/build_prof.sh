#!/bin/bash
# Profiling variant of libopx.so (attention-backward phase stamps compiled in,
# OPX_ATTN_PROF_BUILD=1) at tools/_prof/libopx_prof.so; load it with
# OPX_LIB_PATH=tools/_prof/libopx_prof.so OPX_ATTN_PROF=<cta> (tools/prof_attn_phases.py).
set -e
cd "$(dirname "$0")/../paper_2508_02317_b200/csrc"
make -s -j
PY_SITE=$(python -c "import sysconfig;print(sysconfig.get_paths()['purelib'])")
NCCL=$PY_SITE/nvidia/nccl
mkdir -p ../../tools/_prof
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC --expt-relaxed-constexpr -DOPX_ATTN_PROF_BUILD=1 \
  -I$PY_SITE/include/cudnn_frontend/thirdparty/nlohmann -I$NCCL/include -I../../include \
  -c kernels/attention_bwd_tc.cu -o ../../tools/_prof/attention_bwd_tc.o
OBJS=$(find ../../build/obj -name '*.o' ! -name 'attention_bwd_tc.o')
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/_prof/libopx_prof.so \
  $OBJS ../../tools/_prof/attention_bwd_tc.o -L$NCCL/lib -l:libnccl.so.2 -Xlinker -rpath=$NCCL/lib
echo built tools/_prof/libopx_prof.so
