#!/bin/bash
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sweeps.py tests/test_gpu_sitebuffer.py -q -p no:cacheprovider > gpurun_out/pytest_ds2.log 2>&1
echo "pytest=$?" >> gpurun_out/status.txt
python -c "
import torch, numpy as np
from paper_1309_0551_b200 import _lib, sweeps, inputs
from paper_1309_0551_b200.lattice import Field, Lattice4D
lat=Lattice4D(64,64,64,16); dev=torch.device('cuda',0); g=torch.Generator(device=dev); g.manual_seed(1)
U=Field.from_aos(lat,'mat4',inputs.random_links_torch(lat.volume,4,torch.float32,dev,g))
v=Field.from_aos(lat,'vec',inputs.random_vectors_torch(lat.volume,None,torch.float32,dev,g))
a=sweeps.dslash(U,v,0); print(_lib.last_kernel())
full=sweeps.nn_sweep(U,v).numpy(); got=a.numpy()
from oracle import sweeps as OS
m=OS.parity_mask((64,64,64,16)); print('bitwise', np.array_equal(got[m], full[m]), 'untouched', not np.any(got[~m]))
" > gpurun_out/ds_check.log 2>&1
bash tools/gpu_ab_var.sh "X=1|--workload dslash --dtype f32" "X=1|--workload dslash --dtype f32 --mode fma" "X=1|--workload nn-weak --dtype f32 --dims 48,48,48,16" "X=1|--workload nn-weak --dtype f32"
