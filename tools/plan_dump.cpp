// Host-only: print the dense-conv plan (conv_dense.cu dense_conv_plan) of
// conv shapes, so parity tests can be aimed at every plan variant the
// benchmarked networks use.  g++ -std=c++17 -I paper_2210_09887_b200/csrc
//   -I include -I /usr/local/cuda/include tools/plan_dump.cpp
//   -L paper_2210_09887_b200 -ldfx_b200 -o /tmp/plan_dump
#include <cstdio>
#include <cstdlib>
#include "kernels.hpp"
int main(int argc, char** argv) {
    for (int i = 1; i + 3 < argc + 0 && i + 3 <= argc - 1; i += 4) {
        const int cin = atoi(argv[i]), cout = atoi(argv[i + 1]), k = atoi(argv[i + 2]), t = atoi(argv[i + 3]);
        dfx::DenseConvPlan p = dfx::dense_conv_plan(cin, cout, k, t, 34, 34, (size_t)256 << 20);
        printf("cin=%d cout=%d k=%d t=%d ok=%d KC=%d NBD=%d nNB=%d nbuf=%u nstw=%d nmma=%d npb=%d tpu=%d smax=%d smem=%zu\n",
               cin, cout, k, t, (int)p.ok, p.KC, p.NBD, p.nNB, p.nbuf, p.nstw, p.nmma, p.npb, p.tpu, p.smax, p.smem);
    }
}
