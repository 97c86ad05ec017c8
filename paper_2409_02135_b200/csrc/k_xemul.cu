// k_xemul.cu -- instantiations of k_step_x_emul, the one-GPU concurrent emulation of G ranks running the
// fused statistics exchange (qqa_exchange_emulate; test of the protocol, not a production path).
#define QQA_INST_ONLY
#include "qqa_dispatch.h"

namespace qqa {
template <int M>
XEmulKernel xemul_for(int lanes, int vpl, bool full) {
  if (vpl != 1) return nullptr;
#define QQA_ECASE(L) \
  if (lanes == L) return full ? k_step_x_emul<L, 1, M, true> : k_step_x_emul<L, 1, M, false>;
  QQA_ECASE(1) QQA_ECASE(2) QQA_ECASE(4) QQA_ECASE(8)
#undef QQA_ECASE
  return nullptr;
}

XEmulKernel xemul_kernel(int lanes, int vpl, int mode, bool full) {
  switch (mode) {
    case 0: return xemul_for<0>(lanes, vpl, full);
    case 1: return xemul_for<1>(lanes, vpl, full);
    case 2: return xemul_for<2>(lanes, vpl, full);
    case 3: return xemul_for<3>(lanes, vpl, full);
    case 8: return xemul_for<8>(lanes, vpl, full);
    case 9: return xemul_for<9>(lanes, vpl, full);
    case 10: return xemul_for<10>(lanes, vpl, full);
    case 11: return xemul_for<11>(lanes, vpl, full);
    default: return nullptr;
  }
}
}  // namespace qqa
