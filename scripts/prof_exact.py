import sys; sys.path.insert(0,'/root/repo')
import numpy as np
from paper_2507_04610_b200 import anyq, _abi
rng=np.random.default_rng(1)
w=rng.standard_normal((4096,4096),dtype=np.float32); x=rng.standard_normal((1,4096),dtype=np.float32)
c=_abi.default_config(codebook=_abi.CB_ANY, max_iters=3)
qt=anyq.quantize_any(w,c)
print(anyq.bench_gemm(1, qt, None, x, 3))
