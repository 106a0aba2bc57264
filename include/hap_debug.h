/*
 * hap_debug.h — development aids of libhap.so (profiling experiments, not part of the
 * hot-path boundary of include/hap.h).  Same conventions as hap.h.
 */
#ifndef HAP_DEBUG_H
#define HAP_DEBUG_H

#include "hap.h"

#ifdef __cplusplus
extern "C" {
#endif

/* enable >= 3 in hap_profile: K1 records a timestamp after each of its phases; this returns
 * the phase durations (us, [host] double[7]) of the last hap_align (synchronises). */
HAP_API hap_status hap_profile_k1_phases(hap_ctx ctx, double* us);
/* Development build only (-DHAP_EXPERIMENTS, HAP_K3_EXPERIMENT bit 16 in the environment):
 * K3 globaltimer stamps [sm_count][8 units][8 events]; copies up to n int64 into out [host].
 * HAP_E_INVALID_ARG when none were recorded. */
HAP_API hap_status hap_debug_k3_stamps(hap_ctx ctx, long long* out, int64_t n);
/* Profiling level 3: raw K1 timestamps, [8] kernel phases of CTA 0 then [grid][8] per-CTA
 * events (entry, P1 done, barrier passed, -, P3 done, P4 coefficients done, P4 done, exit);
 * out holds n int64 (at most 8 + 8 * SM count are written). */
HAP_API hap_status hap_debug_k1_stamps(hap_ctx ctx, long long* out, int64_t n);
/* Checked build only (libhap_checked.so, -DHAP_DEVICE_CHECKS):
 * synchronises the device, then writes to *word [host] the first failed device-side bounds /
 * invariant check since the last call ({translation unit << 32 | source line}: 1 k_align.cu,
 * 2 k_perm.cu, 3 k_maskgemm.cu, 4 k_gram.cu; 0 = none) and clears it; it also verifies
 * the guard bytes (0xA5) past the requested size of every workspace buffer of ctx and its
 * batch sub-contexts and returns HAP_E_CUDA (message: the buffer) if one was overwritten.
 * The release library writes 0 and returns HAP_E_INVALID_ARG (no checks compiled in). */
HAP_API hap_status hap_debug_check_status(hap_ctx ctx, uint64_t* word);
/* K3 form of the last test hap_permtest planned on ctx (host value, no sync): *gram = 1 for
 * the Gram form, 0 for the plane form, -1 before any test; the
 * parity tests use it to mirror the kernel's error bound (R14). */
HAP_API hap_status hap_debug_last_form(hap_ctx ctx, int32_t* gram);
/* Scheduling experiments: enqueue a register-only Philox loop of `iters` rounds on
 * ctas x threads threads, no shared memory. */
HAP_API hap_status hap_debug_alu_burn(hap_ctx ctx, uint32_t iters, int ctas, int threads, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HAP_DEBUG_H */
