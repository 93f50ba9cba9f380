// round_plan.h: the per-query plan of the scan rounds of one nn1 batch (R9, R10). Pure host logic
// (no CUDA calls), so the CPU tests drive it through isax_debug_plan_round.
//
// A round scans one query's band (lo, hi] of LB^2 over the sorted positions [plo, phi). After it:
//  - near-list overflow (R9): the caller grows the list and the query starts over (band reset);
//  - candidate-list overflow: the band shrinks to the largest prefix of its 64-bin LB histogram
//    that fits 9/10 of the capacity; when the histogram cannot split it (the first bin alone
//    overflows three times in a row, the band is narrower than 2^-16 of its bounds, or the shrunk
//    edge rounds onto either end of the band) the positions are halved instead, and a completed position
//    range is followed by the next one, twice as long;
//  - otherwise the band is done; if it was capped below the BSF, the next band (hi, +inf) follows.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>

#include "isax_internal.cuh"

namespace isax {

struct RoundState {
    Band band;
    uint32_t plen;    // position mode: length of the next range
    uint32_t nfirst;  // consecutive overflows whose first histogram bin alone overflowed
};

enum PlanAction { PLAN_DONE = 0, PLAN_AGAIN = 1, PLAN_RESCAN = 2, PLAN_ERROR = -1 };

// tused: the threshold the round used (min(band.hi, bsf^2 (1 + delta)) at its start);
// bsf_lim: bsf^2 (1 + delta) now; hist: the round's HIST_BINS counts (read only on overflow)
inline int plan_next_round(RoundState &st, uint32_t cnt, uint32_t cap, const uint32_t *hist, bool near_ovf,
                           float tused, float bsf_lim, uint32_t NP) {
    const float INF = std::numeric_limits<float>::infinity();
    Band &bd = st.band;
    if (cnt <= cap) st.nfirst = 0;
    if (near_ovf) {  // start over with the BSF kept (the caller grows the near list)
        bd = Band{-1.0f, INF, 0u, NP};
        st.plen = NP;
        return PLAN_RESCAN;
    }
    if (cnt > cap) {
        const float lo0 = std::fmax(bd.lo, 0.0f), span = tused - lo0;
        uint64_t cum = 0;
        int kk = -1;
        for (uint32_t bb = 0; bb < HIST_BINS; bb++) {
            cum += hist[bb];
            if (cum > (uint64_t)cap * 9 / 10) break;
            kk = (int)bb;
        }
        const float hi_new = kk < 0 ? lo0 + span / (float)HIST_BINS : lo0 + span * (float)(kk + 1) / (float)HIST_BINS;
        st.nfirst = kk < 0 ? st.nfirst + 1 : 0;
        // (the shrunk edge must lie strictly inside (lo0, tused): in a band a few ulps wide it can
        // round onto either end, and an edge equal to tused would repeat the same round for ever)
        const bool stuck = (kk < 0 && (st.nfirst >= 3 || !(span > std::fmax(lo0, tused) * 1.52587890625e-05f))) ||
                           !(hi_new > lo0) || !(hi_new < tused);
        if (stuck || bd.phi - bd.plo < NP) {
            const uint32_t len = bd.phi - bd.plo;
            if (len <= 1) return PLAN_ERROR;
            bd.phi = bd.plo + len / 2;
            st.plen = len / 2;
        } else {
            bd.hi = hi_new;
        }
        return PLAN_AGAIN;
    }
    if (bd.phi < NP || bd.plo > 0) {  // a position range of a split band completed
        if (bd.phi < NP) {
            const uint64_t len = std::min<uint64_t>(2ull * st.plen, NP);
            st.plen = (uint32_t)len;
            bd.plo = bd.phi;
            bd.phi = (uint32_t)std::min<uint64_t>((uint64_t)bd.plo + len, NP);
            return PLAN_AGAIN;
        }
        bd.plo = 0;  // the band is complete over all positions
        bd.phi = NP;
        st.plen = NP;
    }
    if (tused == bd.hi && bsf_lim > bd.hi) {  // capped below the BSF: the next band
        bd = Band{bd.hi, INF, 0u, NP};
        return PLAN_AGAIN;
    }
    return PLAN_DONE;
}

}  // namespace isax
