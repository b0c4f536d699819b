bash tools/dev/gpu_ab_dirs.sh indexer_gemm _exp_s0x00u _exp_s0x01u _exp_s0x11u _exp_s0x55u
for m in 0x11u 0x55u; do VSP_ROOT=_exp_s$m timeout 300 python -c "
import os,sys; sys.path.insert(0, os.environ['VSP_ROOT'])
import torch, paper_2603_04460_b200 as vsp, oracle, numpy as np
print(vsp.lib_path)
" ; done
