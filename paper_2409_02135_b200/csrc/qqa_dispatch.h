// qqa_dispatch.h -- kernel pointers of the template kernels, one translation unit per step
// mode (k_mode0..3.cu) and one for the K-ary kernels (k_kary.cu), so the library compiles in
// parallel. Only plain host functions cross translation units (no extern kernel templates).
#pragma once
#include "qqa_kernels.cuh"

namespace qqa {
using StepKernel = void (*)(const StepParams);
using RunKernel = void (*)(const RunParams);
using XStepKernel = void (*)(const StepParams, const XParams);
using StepKKernel = void (*)(const StepKParams);
using InitKKernel = void (*)(const InitKParams);
using PackKKernel = void (*)(const float*, uint8_t*, int, int, int);

// k_step<lanes, vpl, MODE> and k_run<lanes, vpl, MODE, cta> (cta 1024 only for vpl 1); nullptr if
// no kernel exists for (lanes, vpl). MODE bit 2 (printed clique) has no k_run.
StepKernel step_kernel_m0(int lanes, int vpl, bool full);
StepKernel step_kernel_m1(int lanes, int vpl, bool full);
StepKernel step_kernel_m2(int lanes, int vpl, bool full);
StepKernel step_kernel_m3(int lanes, int vpl, bool full);
StepKernel step_kernel_m4(int lanes, int vpl, bool full);
StepKernel step_kernel_m5(int lanes, int vpl, bool full);
StepKernel step_kernel_m6(int lanes, int vpl, bool full);
StepKernel step_kernel_m7(int lanes, int vpl, bool full);
StepKernel step_kernel_m8(int lanes, int vpl, bool full);    // 8-11: weighted graphs (+ clamp / noise)
StepKernel step_kernel_m9(int lanes, int vpl, bool full);
StepKernel step_kernel_m10(int lanes, int vpl, bool full);
StepKernel step_kernel_m11(int lanes, int vpl, bool full);
RunKernel run_kernel_m0(int lanes, int vpl, int cta, bool full);
RunKernel run_kernel_m1(int lanes, int vpl, int cta, bool full);
RunKernel run_kernel_m2(int lanes, int vpl, int cta, bool full);
RunKernel run_kernel_m3(int lanes, int vpl, int cta, bool full);
RunKernel run_kernel_m4(int lanes, int vpl, int cta, bool full);   // nullptr: modes 4-7 run launch-per-step
RunKernel run_kernel_m5(int lanes, int vpl, int cta, bool full);
RunKernel run_kernel_m6(int lanes, int vpl, int cta, bool full);
RunKernel run_kernel_m7(int lanes, int vpl, int cta, bool full);
RunKernel run_kernel_m8(int lanes, int vpl, int cta, bool full);
RunKernel run_kernel_m9(int lanes, int vpl, int cta, bool full);
RunKernel run_kernel_m10(int lanes, int vpl, int cta, bool full);
RunKernel run_kernel_m11(int lanes, int vpl, int cta, bool full);

// k_step_st<lanes, MODE> (staged state, VPL = 1, FULL shapes), MODE 0..3; nullptr otherwise.
StepKernel stage_kernel_m0(int lanes);
StepKernel stage_kernel_m1(int lanes);
StepKernel stage_kernel_m2(int lanes);
StepKernel stage_kernel_m3(int lanes);

// k_step_x<lanes, vpl, MODE> (fused statistics exchange), MODE 0..3 and 8..11 (weighted); nullptr otherwise.
XStepKernel xstep_kernel_m0(int lanes, int vpl, bool full);
XStepKernel xstep_kernel_m1(int lanes, int vpl, bool full);
XStepKernel xstep_kernel_m2(int lanes, int vpl, bool full);
XStepKernel xstep_kernel_m3(int lanes, int vpl, bool full);
XStepKernel xstep_kernel_m8(int lanes, int vpl, bool full);
XStepKernel xstep_kernel_m9(int lanes, int vpl, bool full);
XStepKernel xstep_kernel_m10(int lanes, int vpl, bool full);
XStepKernel xstep_kernel_m11(int lanes, int vpl, bool full);
// k_step_xs<lanes, vpl, MODE> (owner-slotted exchange), the same modes; nullptr otherwise.
XStepKernel xsstep_kernel_m0(int lanes, int vpl, bool full);
XStepKernel xsstep_kernel_m1(int lanes, int vpl, bool full);
XStepKernel xsstep_kernel_m2(int lanes, int vpl, bool full);
XStepKernel xsstep_kernel_m3(int lanes, int vpl, bool full);
XStepKernel xsstep_kernel_m8(int lanes, int vpl, bool full);
XStepKernel xsstep_kernel_m9(int lanes, int vpl, bool full);
XStepKernel xsstep_kernel_m10(int lanes, int vpl, bool full);
XStepKernel xsstep_kernel_m11(int lanes, int vpl, bool full);

// k_step_x_emul<lanes, 1, MODE> (one-GPU concurrent emulation of the fused exchange, k_xemul.cu):
// lanes 1..8, vpl 1, MODE 0..3 and 8..11; nullptr otherwise.
using XEmulKernel = void (*)(const XEmulParams);
XEmulKernel xemul_kernel(int lanes, int vpl, int mode, bool full);

// k_run_cluster<MODE> (MODE 0..3, compiled in k_cluster.cu); nullptr otherwise.
RunKernel cluster_kernel(int mode);

// Segmented gather (k_seg.cu): k_seg_gather<lanes, FIRST> and k_step_seg<lanes, MODE> for VPL 1, FULL
// shapes, MODE 0..3; false otherwise.
bool seg_kernels(int lanes, int mode, StepKernel& first, StepKernel& mid, StepKernel& last);

// K-ary kernels for KP in {4, 8, 12, 16}; false otherwise.
bool kary_kernels(int KP, int K, int mode, StepKKernel& ks, InitKKernel& ki, PackKKernel& kp);
// k_step_Kq<KP, MODE> (colour quads, KP = 12 / 16); nullptr otherwise.
StepKKernel kary_quad_kernel(int KP, int mode);
int kary_quad_reps(int KP);   // replicas per warp of kary_quad_kernel(KP)
}  // namespace qqa
