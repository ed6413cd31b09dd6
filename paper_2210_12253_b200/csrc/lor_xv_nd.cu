// lor_xv_nd.cu -- Nedelec instantiations of the extended-frame vector-space kernels (lor_xv.cuh).
// four cell corners between compiler fences in the ND cell routine (more ILP in the cell phase of
// k_xv_fill; C4 fill 3.23 -> 3.18 ms; the element pass keeps one at a time)
#define ND_FENCE 4
// and the next-residency CTA's row pointers / positions prefetched into L2 (C4 fill 3.18 -> 3.15 ms;
// RT is slower with it: 0.90 -> 1.00 ms)
#define XV_PF_ROWS 1
#include "lor_xv.cuh"

namespace lorb {

cudaError_t xv_run_nd(int what, int p, const XvArgs &a, cudaStream_t st) { return run_sp<SP_ND>(what, p, a, st); }
int xv_supported_nd(int p, const int cmax[3]) { return p >= 1 && p <= 8 ? supported_sp<SP_ND>(p, cmax) : 0; }
int64_t xv_words_nd(int p, const int cmax[3]) { return p >= 1 && p <= 8 ? words_sp<SP_ND>(p, cmax) : 0; }

}  // namespace lorb
