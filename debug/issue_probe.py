import ctypes as C, torch
lib = C.CDLL("debug/libissueprobe.so")
for g in (1, 2, 4, 5):
    out = torch.zeros(2 * g, dtype=torch.int64, device="cuda")
    it = 2000
    lib.run(C.c_void_p(out.data_ptr()), g, it)
    v = out.cpu().numpy().reshape(g, 2)
    print(f"{g} issuing warps: issue {v[:, 0].mean() / it:.0f} cycles/batch, round trip {v[:, 1].mean() / it:.0f} cycles/batch "
          f"(pipe-bound would be {g * 6 * 56} per batch)")
