import ctypes as C, torch
lib = C.CDLL("debug/libcta2probe.so")
torch.manual_seed(0)
A = (torch.randn(256, 16) * 0.5).half().cuda()
B = (torch.randn(96, 16) * 0.5).half().cuda()
D = torch.zeros(256, 96, device="cuda")
rc = lib.run_probe(C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()), C.c_void_p(D.data_ptr()))
ref = A.float() @ B.float().T
print("rc", rc, "max err", (D - ref).abs().max().item(), "ref max", ref.abs().max().item())
# which B rows did each CTA use? try the alternative hypothesis too

for cg2 in (0, 1):
    for ncl in (1, 74):
        cyc = torch.zeros(2 * ncl, dtype=torch.int64, device="cuda")
        n = 2000
        rc = lib.run_tput(cg2, C.c_void_p(cyc.data_ptr()), n, ncl)
        v = cyc.cpu().numpy()
        v = v[v > 0]
        print(f"cta_group::{2 if cg2 else 1} clusters={ncl}: {v.mean() / n:.1f} cycles per MMA (M={256 if cg2 else 128}, N=96, K=16)")
out = torch.zeros(2, dtype=torch.int64, device="cuda")
it = 2000
lib.run_pingpong(C.c_void_p(out.data_ptr()), it)
print(f"cluster mbarrier round trip: {out.cpu().numpy()[0] / it:.0f} cycles (one-way ~half)")
