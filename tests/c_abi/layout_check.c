/* Plain-C client of include/hpz.h: proves the header is C (not C++) and the library links
 * from C.  Host-only context (device -1): layout queries, no GPU needed.  Prints the layout
 * of BASELINE's Falcon-7B decoder block at P=8, P'=4 and exits 0 iff it matches Eq. (1) with
 * the R2 padding (207,071,232 / 25,883,904 / 51,767,808). */
#include <stdio.h>

#include "hpz.h"

int main(void) {
  hpz_ctx* ctx = NULL;
  if (hpz_init(8, 4, 3, -1, &ctx) != HPZ_OK) return 2;
  const int64_t numel[2] = {207070080, 4544 * 2};
  uint64_t arena = 0;
  if (hpz_register_flat_params(ctx, 2, numel, HPZ_BF16, 256, 2, &arena) != HPZ_OK) return 3;
  hpz_layer_info_t info;
  if (hpz_layer_info(ctx, 0, &info) != HPZ_OK) return 4;
  printf("numel_pad=%lld shard=%lld sec_shard=%lld arena=%llu version=%d\n", (long long)info.numel_pad,
         (long long)info.shard, (long long)info.sec_shard, (unsigned long long)arena, hpz_version());
  int ok = info.numel_pad == 207071232 && info.shard == 25883904 && info.sec_shard == 51767808;
  if (hpz_set_order(ctx, 7, 0, 0) != HPZ_EINVAL) ok = 0;       /* invalid order rejected */
  if (hpz_fwd_gather(ctx, 0, (void*)0x1000, NULL) != HPZ_ESTATE) ok = 0;   /* no arena bound */
  hpz_finalize(ctx);
  return ok ? 0 : 1;
}
