import ctypes as C, os, sys, time
lib = C.CDLL(os.path.join(os.environ.get("GRAFT_REPO_ROOT","/root/repo"), "paper_2604_17861_b200/lib/libgpuos_bench.so"))
lib.gb_config5.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
out = (C.c_double * 8)()
s, n, w = (int(x) for x in sys.argv[1:4])
t0 = time.time()
lib.gb_config5(0, s, n, w, out)
print(s, n, w, "tasks/s", out[0], "GB/s", out[1], "failed", out[2], "slow ms", out[3], "wall", time.time() - t0, flush=True)
