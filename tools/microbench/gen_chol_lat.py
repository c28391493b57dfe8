"""Regenerates chol_lat.cu: chol_inv_regs copied out of factor.cu into a standalone clock64 timer."""
import os
import re

here = os.path.dirname(os.path.abspath(__file__))
src = open(os.path.join(here, "..", "..", "paper_1703_09074_b200", "csrc", "factor.cu")).read()
a = src.index("template <int KR, int KC>\n__device__ void chol_inv_regs")
b = src.index("template <int KR, int KC>\n__device__ void sign_reconstruct_regs")
c = src.index("__device__ void sign_reconstruct(double* G, int n, int ld, int rows, double* sgn) {\n  const int nw")
t = open(os.path.join(here, "chol_lat.cu")).read()
head, tail = t.split("template <int KR, int KC>\n__global__ void run", 1)
head = head[: head.index("template <int KR, int KC>")]
open(os.path.join(here, "chol_lat.cu"), "w").write(head + src[a:c] + "template <int KR, int KC>\n__global__ void run" + tail)
