mkdir -p gpurun_out/r2
V=$PWD/paper_2308_07173_b200/variants
timeout 300 python tools/debug_bits.py /tmp/b_new.npy > gpurun_out/r2/bits_new.log 2>&1
GICP_LIB_VARIANT=$V/libgicp_head2.so timeout 300 python tools/debug_bits.py /tmp/b_head.npy > gpurun_out/r2/bits_head.log 2>&1
python -c "
import numpy as np
a=np.load('/tmp/b_new.npy'); b=np.load('/tmp/b_head.npy')
for k in range(len(a)):
    d = np.flatnonzero(a[k] != b[k]); print(k, 'differ at', d, a[k][d], b[k][d])
A=np.load('/tmp/b_new_align.npy'); B=np.load('/tmp/b_head_align.npy'); print('align', np.abs(A-B).max())
" > gpurun_out/r2/bits_cmp.log 2>&1
