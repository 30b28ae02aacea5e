/*
 * autobyte_testing.h — test hooks of libautobyte.so (not part of the product API; the tests call
 * them to exercise multi-rank protocols on a single GPU).
 */
#ifndef AUTOBYTE_TESTING_H_
#define AUTOBYTE_TESTING_H_

#include "autobyte.h"

#ifdef __cplusplus
extern "C" {
#endif

/* The NVLink peer-memory key exchange (exchange.cu) among G virtual ranks on the
 * ctx's ONE device: G windows laid out like the IPC-shared ones, virtual rank r runs the same
 * kernel (push its keys into every window, raise its epoch flag everywhere, wait for all G flags,
 * reduce) on its own stream with one block, `calls` times in a row (epochs 1..calls, both window
 * parities). keys: DEVICE [G][2J] u64 (rank r's autobyte_argmax_keys output); outputs DEVICE [G][J]
 * each: what virtual rank r returns from the last call. absent_rank (0..G-1, or -1 for none) is
 * never launched, so the others wait for it until timeout_ms and the call returns AB_E_NCCL (the
 * status-word path of a dead peer). 1 <= G <= 8, J >= 1, calls >= 1, timeout_ms >= 1 (else
 * AB_E_SHAPE). Synchronous. */
autobyte_status autobyte_debug_peer_loopback(autobyte_ctx* ctx, int32_t G, int32_t J, int32_t calls,
                                             int32_t absent_rank, int32_t timeout_ms, const uint64_t* keys,
                                             int32_t* best_idx, float* best_score, float* cur_score);

/* Memory debugging (the pool has no compute-sanitizer). With AUTOBYTE_DEBUG_MEM=1 set when a ctx is
 * created, every library allocation from then on is filled with 0xFF bytes (NaN as fp32) so reads of
 * never-written workspace surface as NaN / garbage in parity checks, and carries a 256-byte 0xA5
 * canary after its requested size. This call synchronises the ctx's device and returns how many
 * live canaries of that device were overwritten (0 = none; -1 on a CUDA error or NULL ctx). */
int32_t autobyte_debug_mem_check(autobyte_ctx* ctx);

/* The library's fast 32-bit division (K2's per-tile index splits: tile -> (job, tile of job) by
 * tiles_per_job, candidate -> (p, q) by Q): the host-built multiplier / shift applied on the host,
 * out[i] = n[i] / d for 0 <= n[i] < 2^31, d >= 1 (else AB_E_SHAPE). Host memory, no GPU needed. */
autobyte_status autobyte_debug_fastdiv(uint32_t d, const uint32_t* n, int32_t count, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif /* AUTOBYTE_TESTING_H_ */
