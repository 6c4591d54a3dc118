// ig_internal.h — libig functions shared between its translation units (not part of the ABI).
#pragma once
#include "../../include/ig.h"
#include "../../include/ig_ops.h"

// a1 on a host bitmap for a grid of L tokens (ig_mask_build_host without a model context); W =
// grid width in tokens and row_bytes = one K/V row, for the copy lane's DMA grouping (0: unknown)
ig_status ig_mask_build_host_L(int device, int L, const uint8_t* mask, void* stream, ig_mask** out, int* n_masked,
                               int W = 0, int row_bytes = 0);
// set the thread-local message returned by ig_last_error() (other translation units' errors)
ig_status ig_internal_err(ig_status s, const char* msg);
// the process-wide tuning struct (ig_tuning_get/set; seeded from the environment on first use)
const ig_tuning& ig_tuning_ref();
