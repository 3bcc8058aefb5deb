import ctypes as C, torch
lib = C.CDLL("debug/libcpprobe.so")
# src: 8 planes x 128 lanes x 4 fp32: value = lane*100 + channel
src = torch.zeros(8, 128, 4)
for g in range(8):
    for l in range(128):
        for k in range(4):
            src[g, l, k] = l * 100 + 4 * g + k
src = src.cuda().contiguous()
out = torch.zeros(128, 32, device="cuda")
for plane in (2048, 2176):
    out.zero_()
    rc = lib.run_probe(C.c_void_p(src.data_ptr()), C.c_void_p(out.data_ptr()), plane)
    want = torch.arange(128, device="cuda")[:, None] * 100 + torch.arange(32, device="cuda")[None, :]
    ok = torch.equal(out, want.float())
    print("plane", plane, "rc", rc, "match", ok)
    if not ok:
        print(out[:3, :16].tolist())
        print(out[8:10, :16].tolist())
