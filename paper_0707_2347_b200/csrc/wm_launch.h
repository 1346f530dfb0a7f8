// Launch-attribute switches shared by every kernel launcher.
#pragma once

namespace wm {
// Programmatic dependent launch on every kernel (default on; the "pdl" context
// option turns it off for measurements).
extern bool g_pdl;
// launch shapes of the frame prep / combine (wm_frame.cu; context options
// "prep_rows", "comb_block")
extern int g_prep_rows;
extern unsigned g_comb_block;
}  // namespace wm

// INVARIANT (the early loads of wm_frame.cu rely on it, wm_runtime.cu
// mark_early_loads): every kernel executes griddepcontrol.wait BEFORE it triggers
// its dependents (WM_PDL_EARLY_* / WM_PDL_LATE_* come after the wait; a kernel
// without a trigger releases them when it exits).  A dependent's code ahead of
// its own wait therefore runs only after everything its direct predecessors
// waited for has completed.
//
// Where a kernel lets its programmatic dependents launch.  A dependent launched
// early parks its CTAs at griddepcontrol.wait on the SMs the running kernel
// uses; for compute-bound kernels that costs issue slots (measured: the float64
// DMMA leaf chain of config 5 ran 1.8x slower), so those trigger after their
// main loop.  0 = right after griddepcontrol.wait, 1 = late.
#ifndef WM_PDL_LATE_COMPUTE
#define WM_PDL_LATE_COMPUTE 1
#endif
#ifndef WM_PDL_LATE_MEMORY
#define WM_PDL_LATE_MEMORY 0
#endif
// Measurement timeline (the "trace" context option, wm_diag_trace): thread 0 of
// every CTA folds %globaltimer into its launch's [first start, last end] slot.
#define WM_TL_NOW(t_) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_))
#define WM_TL_BEGIN(tl)                                       \
    do {                                                      \
        if ((tl) && threadIdx.x == 0) {                       \
            unsigned long long t_;                            \
            WM_TL_NOW(t_);                                    \
            atomicMin((tl), t_);                              \
        }                                                     \
    } while (0)
#define WM_TL_END(tl)                                         \
    do {                                                      \
        if ((tl) && threadIdx.x == 0) {                       \
            unsigned long long t_;                            \
            WM_TL_NOW(t_);                                    \
            atomicMax((tl) + 1, t_);                          \
        }                                                     \
    } while (0)
#define WM_PDL_TRIGGER() asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory")
#if WM_PDL_LATE_COMPUTE
#define WM_PDL_EARLY_C()
#define WM_PDL_LATE_C() WM_PDL_TRIGGER()
#else
#define WM_PDL_EARLY_C() WM_PDL_TRIGGER()
#define WM_PDL_LATE_C()
#endif
#if WM_PDL_LATE_MEMORY
#define WM_PDL_EARLY_M()
#define WM_PDL_LATE_M() WM_PDL_TRIGGER()
#else
#define WM_PDL_EARLY_M() WM_PDL_TRIGGER()
#define WM_PDL_LATE_M()
#endif
