import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_0909_2000_b200 import _native, datagen
L = _native.lib(); ctx = ctypes.c_void_p(); assert L.ap_ctx_create(0, ctypes.byref(ctx)) == 0
w, r, rows = 2048, 1, 1184
x = datagen.uniform(7, 0, w + rows - 1, datagen.DNA); y = datagen.uniform(7, 1, 40000, datagen.DNA)
cfg = _native.ApConfig(window_w=w, step_h=1, blowup_r=r, has_threshold=0, threshold_half=0, n_devices=1, row_begin=0, row_end=0)
dx, dy = torch.from_numpy(x.copy()).cuda(), torch.from_numpy(y.copy()).cuda()
out = torch.empty(rows * (y.size - w + 1), dtype=torch.int16, device="cuda")
assert L.ap_ctx_plot_dense_device(ctx, dx.data_ptr(), x.size, dy.data_ptr(), y.size, ctypes.byref(cfg), out.data_ptr(), None) == 0
print("ok", L.ap_ctx_last_kernel_ms(ctx))
