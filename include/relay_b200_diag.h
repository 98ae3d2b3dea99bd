/*
 * relay_b200_diag -- diagnostics-only entry points.
 *
 * Exported by librelay_b200_diag.so (the same kernels built with
 * -DRB_DIAG=1, paper_2402_14808_b200/build.py), never by the production
 * librelay_b200.so: layout probes and per-CTA timestamp instrumentation used
 * by tests/test_gpu_parity.py::test_umma_probe_layouts and profiles/diag_*.py.
 * Same conventions as relay_b200.h.
 */
#ifndef RELAY_B200_DIAG_H
#define RELAY_B200_DIAG_H

#include "relay_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/*
 * Probe of the tcgen05 operand layouts used by rb_system_attention (one
 * CTA): S^T = K.Q^T and O^T = V^T.P^T for K,V [128][128], Q [nq][128],
 * P [nq][128] bf16 -> s_out, o_out fp32 [128][nq].
 */
int rb_debug_umma_probe(const void* k, const void* q, const void* v, const void* p, int nq,
                        float* s_out, float* o_out, void* stream);

/*
 * When `buf` (device, [grid][8] u64) is non-NULL, subsequent launches record
 * per-CTA %globaltimer stamps into it (system kernel: entry, prologue done,
 * first S tile, group ends, producer ends, exit; context kernel after 1024 x 8
 * slots).  NULL disables.  Not thread-safe: process-global state.
 */
int rb_debug_set_timestamps(void* buf);

#ifdef __cplusplus
}
#endif
#endif /* RELAY_B200_DIAG_H */
