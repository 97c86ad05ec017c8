// k_kary.cu -- the K-ary (graph colouring, NEXT-4) kernel instantiations.
#define QQA_INST_ONLY
#include "qqa_dispatch.h"

namespace qqa {
bool kary_kernels(int KP, int K, int mode, StepKKernel& ks, InitKKernel& ki, PackKKernel& kp) {
  const bool noise = (mode & kModeNoise) != 0;
  const bool fk = K == KP;   // no padding colours: k_step_K<KP, MODE, true>
#define QQA_KCASE(KPV)                                            \
  if (KP == KPV) {                                                \
    ks = noise ? (fk ? k_step_K<KPV, kModeNoise, true> : k_step_K<KPV, kModeNoise>)         \
               : (fk ? k_step_K<KPV, 0, true> : k_step_K<KPV, 0>);                         \
    ki = k_init_K<KPV>;                                           \
    kp = k_pack_K<KPV>;                                           \
    return true;                                                  \
  }
  QQA_KCASE(4) QQA_KCASE(8) QQA_KCASE(12) QQA_KCASE(16)
#undef QQA_KCASE
  return false;
}

StepKKernel kary_quad_kernel(int KP, int mode) {
  const bool noise = (mode & kModeNoise) != 0;
  if (KP == 8) return noise ? k_step_Kq<8, kModeNoise> : k_step_Kq<8, 0>;
  if (KP == 12) return noise ? k_step_Kq<12, kModeNoise> : k_step_Kq<12, 0>;
  if (KP == 16) return noise ? k_step_Kq<16, kModeNoise> : k_step_Kq<16, 0>;
  return nullptr;
}

int kary_quad_reps(int KP) { return KP == 8 ? quad_reps<8>() : quad_reps<16>(); }
}  // namespace qqa
