// k_mode6.cu -- k_step of step mode 6 (bit 0 clamp, bit 1 Langevin noise, bit 2 printed clique).
#include "k_mode.cuh"

namespace qqa {
StepKernel step_kernel_m6(int lanes, int vpl, bool full) { return step_for<6>(lanes, vpl, full); }
RunKernel run_kernel_m6(int lanes, int vpl, int cta, bool full) { return run_kernel_for<6>(lanes, vpl, cta, full); }
}  // namespace qqa
