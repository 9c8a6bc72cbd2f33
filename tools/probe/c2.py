import ctypes as C, os, sys
lib = C.CDLL(os.path.join(os.environ.get("GRAFT_REPO_ROOT","/root/repo"), "paper_2604_17861_b200/lib/libgpuos_bench.so"))
lib.gb_config2.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
out = (C.c_double * 16)()
lib.gb_config2(0, int(os.environ.get("C2_TASKS", "20000")), 2, out)
print(os.environ.get("TAG",""), "tasks/s %.0f GB/s %.1f bytes/task %.0f failed %d submit ns %.0f" % (out[0], out[1], out[3], out[4], out[5]), flush=True)
