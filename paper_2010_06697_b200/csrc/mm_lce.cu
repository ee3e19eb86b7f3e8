// Liquid-crystal-elastomer local step and frozen Frank force (placeholder).
#include "mm_internal.cuh"

int mm_run_lce(mm_ctx *ctx, double, double, int64_t, int, mm_local_stats *) {
    return mm_fail(ctx, MM_ERR_CONFIG, "LCE local step not built yet");
}

int mm_run_frozen(mm_ctx *ctx) {
    return mm_fail(ctx, MM_ERR_CONFIG, "LCE frozen data not built yet");
}
