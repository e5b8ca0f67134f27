// osim_exh_impl.cuh -- instantiations of the prefix-sharing exhaustive kernel
// for one (DMA, sigma-is-a-power-of-two) combination.  Included by
// osim_exh_d2s1.cu / osim_exh_d2s0.cu / osim_exh_d1.cu with OSIM_DMA, OSIM_SP2
// and OSIM_EXH_NAME defined.
#include "osim_launch.cuh"

namespace osim {
namespace {

template <int N, int L>
int exh_t(const LaunchCfg& cfg, const double* d_durs, double sigma, uint64_t lo, uint64_t hi, double thr,
          Part* parts, int max_parts, double* d_ms, int* grid_out, osim_summary* d_out, unsigned long long* d_below,
          unsigned* d_done, unsigned shard, unsigned shards) {
    // makespans out or a positive threshold need the stats variant
    auto k = (d_ms || thr > 0.0) ? k_exhaustive_pfx<N, OSIM_DMA, OSIM_SP2, L, true>
                                 : k_exhaustive_pfx<N, OSIM_DMA, OSIM_SP2, L, false>;
    constexpr uint64_t LF = Fact<L>::v;
    const uint64_t prefixes = (hi + LF - 1) / LF - lo / LF;
    constexpr uint64_t kPer = (uint64_t)kPfxQ * kBlock;
    const uint64_t calls = (prefixes + kPer - 1) / kPer;  // this shard's: calls shard, shard + shards, ...
    const uint64_t mine = calls > shard ? (calls - shard + shards - 1) / shards : 1;
    const uint64_t slots = (uint64_t)cached_ctas_per_sm((const void*)k, kBlock, kPfxDynSmem) * cfg.sms;
    // a shard of at most half the resident CTA slots (C3 at 8 ranks: 148
    // calls) splits every call over two CTAs of 256 prefixes each (one per
    // thread): twice the CTAs for the same partition, half the serial work
    // per thread
    const unsigned split = (2 * mine <= slots) ? 2u : 1u;
    int g = grid_for_sms(k, kBlock, kPfxDynSmem, cfg.sms, mine * split);
    if (g > max_parts) g = max_parts;
    g -= g % (int)split;
    k<<<g, kBlock, kPfxDynSmem, cfg.st>>>(d_durs, sigma, lo, hi, thr, parts, d_ms, d_out, d_below, d_done, shard,
                                          shards, split);
    *grid_out = g;
    return 0;
}

template <int N>
int exh_n(int L, const LaunchCfg& cfg, const double* d_durs, double sigma, uint64_t lo, uint64_t hi,
          double thr, Part* parts, int max_parts, double* d_ms, int* g, osim_summary* o, unsigned long long* b,
          unsigned* dn, unsigned sh, unsigned shs) {
    if constexpr (tunable_n(N)) {
        if (L == 3) return exh_t<N, 3>(cfg, d_durs, sigma, lo, hi, thr, parts, max_parts, d_ms, g, o, b, dn, sh, shs);
        if (L == 5) return exh_t<N, 5>(cfg, d_durs, sigma, lo, hi, thr, parts, max_parts, d_ms, g, o, b, dn, sh, shs);
        if (L == 4) return exh_t<N, 4>(cfg, d_durs, sigma, lo, hi, thr, parts, max_parts, d_ms, g, o, b, dn, sh, shs);
    }
    return exh_t<N, default_pfx_l(N)>(cfg, d_durs, sigma, lo, hi, thr, parts, max_parts, d_ms, g, o, b, dn, sh, shs);
}

}  // namespace

int OSIM_EXH_NAME(int n, int L, const LaunchCfg& cfg, const double* d_durs, double sigma, uint64_t lo,
                  uint64_t hi, double thr, Part* parts, int max_parts, double* d_ms, int* g, osim_summary* d_out,
                  unsigned long long* d_below, unsigned* d_done, unsigned shard, unsigned shards) {
    switch (n) {
#define OSIM_CASE(NN) \
    case NN: return exh_n<NN>(L, cfg, d_durs, sigma, lo, hi, thr, parts, max_parts, d_ms, g, d_out, d_below, d_done, \
                         shard, shards);
        OSIM_CASE(1) OSIM_CASE(2) OSIM_CASE(3) OSIM_CASE(4) OSIM_CASE(5) OSIM_CASE(6)
        OSIM_CASE(7) OSIM_CASE(8) OSIM_CASE(9) OSIM_CASE(10) OSIM_CASE(11) OSIM_CASE(12)
        OSIM_CASE(13) OSIM_CASE(14) OSIM_CASE(15) OSIM_CASE(16)
#undef OSIM_CASE
    }
    return -1;
}

}  // namespace osim
