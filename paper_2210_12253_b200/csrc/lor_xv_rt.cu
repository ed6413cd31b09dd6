// lor_xv_rt.cu -- Raviart-Thomas instantiations of the extended-frame vector-space kernels (lor_xv.cuh).
#include "lor_xv.cuh"

namespace lorb {

cudaError_t xv_run_rt(int what, int p, const XvArgs &a, cudaStream_t st) { return run_sp<SP_RT>(what, p, a, st); }
int xv_supported_rt(int p, const int cmax[3]) { return p >= 1 && p <= 8 ? supported_sp<SP_RT>(p, cmax) : 0; }
int64_t xv_words_rt(int p, const int cmax[3]) { return p >= 1 && p <= 8 ? words_sp<SP_RT>(p, cmax) : 0; }

cudaError_t launch_xv_setup(int space, int p, const XvArgs &a, cudaStream_t st) {
  return space == SP_ND ? xv_run_nd(0, p, a, st) : xv_run_rt(0, p, a, st);
}
cudaError_t launch_xv_sym(int space, int p, const XvArgs &a, cudaStream_t st) {
  return space == SP_ND ? xv_run_nd(1, p, a, st) : xv_run_rt(1, p, a, st);
}
cudaError_t launch_xv_fill(int space, int p, const XvArgs &a, cudaStream_t st) {
  return space == SP_ND ? xv_run_nd(2, p, a, st) : xv_run_rt(2, p, a, st);
}
int xv_supported(int space, int p, const int cmax[3]) {
  return space == SP_ND ? xv_supported_nd(p, cmax) : (space == SP_RT ? xv_supported_rt(p, cmax) : 0);
}
int64_t xv_map_words(int space, int p, const int cmax[3]) {
  return space == SP_ND ? xv_words_nd(p, cmax) : xv_words_rt(p, cmax);
}
int xv_pos_words(int space) { return space == SP_ND ? 12 : 4; }

}  // namespace lorb
