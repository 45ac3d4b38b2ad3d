// K5 — constant-(floor(k)+w) KV cache decode step. (implementation follows)
#include "skb_common.cuh"
#include "skb_internal.h"

struct skb_cache {
    int dummy;
};

extern "C" {
int skb_cache_create(const skb_attn_desc*, skb_cache**) { return SKB_ECONFIG; }
int skb_cache_destroy(skb_cache*) { return SKB_OK; }
int skb_cache_step(skb_cache*, const void*, const void*, const void*, const double*, void*, void*) {
    return SKB_ECONFIG;
}
int skb_cache_state(skb_cache*, int64_t, int32_t*, int64_t*, double*, int64_t*, int64_t*, void*) {
    return SKB_ECONFIG;
}
}

struct skb_stream {
    int dummy;
};
extern "C" {
int skb_stream_create(double, int64_t, int64_t, skb_stream**) { return SKB_ECONFIG; }
int skb_stream_destroy(skb_stream*) { return SKB_OK; }
int skb_stream_push(skb_stream*, const double*, int64_t, double*, uint8_t*, void*) { return SKB_ECONFIG; }
int skb_stream_query(skb_stream*, skb_stream_info*, void*) { return SKB_ECONFIG; }
int skb_stream_survivors(skb_stream*, double*, int64_t*, uint8_t*, void*) { return SKB_ECONFIG; }
}
