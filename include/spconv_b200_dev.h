/*
 * spconv_b200_dev.h -- development entry points of libspconv_b200.so (not
 * part of the drop-in interface; no reference counterpart).
 */
#ifndef SPCONV_B200_DEV_H
#define SPCONV_B200_DEV_H

#include "spconv_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Run FWD/BWI (3x3 stride 1, V=16) with one tile-kernel configuration
 * `variant` instead of the dispatcher's choice (tile_conv.cu
 * launch_tile_conv_variant).  The product build keeps the branch /
 * jump-table configurations the tests compare bit for bit; the tuning
 * tables of tools/tune.py (1x1 and BWW variants included) need the
 * development build (`make -C paper_1911_10175_b200/csrc DEV=1`).  Same
 * validation as spc_sparse_*. */
spc_status spc_debug_conv_variant(int variant, const spc_tensor* src, const spc_tensor* filt, const spc_shape* shape,
                                  const spc_plan* plan, int mode, spc_tensor* dst, spc_counters* d_counters,
                                  void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPCONV_B200_DEV_H */
