// tail.cuh — device-resident coarse levels (placeholder until the cluster kernel lands).
#pragma once
#include "internal.cuh"

static inline bool tail_supported(const mss_ctx*, int) { return false; }
static inline int tail_pcg(mss_ctx*, int) { return MSS_EUNSUPPORTED; }
static inline int tail_setup(mss_ctx*) { return MSS_OK; }
