import ctypes, os, sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_07192_b200 import native
native.LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), os.environ.get("DIAG_LIB", "libpipefill_diag.so"))
native._SIGNATURES["pf_gemm_diag"] = (ctypes.c_int, [ctypes.c_void_p, ctypes.c_int])
from paper_2410_07192_b200 import kernels as K
native.load(native.LIB_PATH)
native.require_device()
lib = native.load()
SHAPES = [(16384, 3072, 1024, False, False), (16384, 1024, 1024, False, True), (16384, 4096, 1024, True, False),
          (16384, 1024, 4096, False, True), (16384, 4096, 1024, False, False), (8192, 8192, 8192, False, False)]
for (m, n, k, gelu, res) in SHAPES:
    x = torch.randn(m, k, device="cuda").bfloat16(); w = (torch.randn(n, k, device="cuda") * k ** -0.5).bfloat16()
    b = torch.randn(n, device="cuda").bfloat16(); y = torch.empty(m, n, device="cuda").bfloat16()
    r = torch.randn(m, n, device="cuda").bfloat16() if res else None
    for _ in range(3): K.linear(x, w, b, gelu=gelu, residual=r, out=y)
    torch.cuda.synchronize()
    lib.pf_gemm_diag(None, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); K.linear(x, w, b, gelu=gelu, residual=r, out=y); e1.record(); torch.cuda.synchronize()
    d = (ctypes.c_ulonglong * 16)()
    lib.pf_gemm_diag(d, 0)
    ms = e0.elapsed_time(e1)
    ghz = d[8] / max(d[9], 1)
    ctas = 74 if os.environ.get("PF_GEMM_PAIR") == "1" else 148
    cyc = ms * 1e-6 * ghz * 1e9 * 148
    flops = 2.0 * m * n * k
    mma_ideal = flops / 2 / ctas / (4096 * (2 if ctas == 74 else 1))
    print(f"{m}x{n}x{k} gelu={gelu} res={res} {ms*1e3:.1f}us {flops/ms/1e9:.0f}TF clk={ghz:.2f}GHz kernel-cyc~{cyc/148:.0f} ideal-mma-cyc/CTA={mma_ideal:.0f} mma-loop-sum/CTA={d[4]/ctas:.0f}  mma_wait_full={d[0]/148:.0f} mma_wait_tempty={d[1]/148:.0f} prod_wait_empty={d[2]/148:.0f} epi_wait_tfull(8 warps)={d[3]/148/8:.0f} | per tile: mma_loop={d[4]/max(d[7],1):.0f} cyc, epi_busy/warp={d[5]/max(d[6],1):.0f} cyc, tiles={d[7]}")
