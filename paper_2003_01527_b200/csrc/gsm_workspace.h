// gsm_workspace.h — per-graph device workspace reused across gsm_match calls
// (grow-only buffers: frontiers, per-row plans, counters), so steady-state
// matches do no device allocation.
#pragma once

#include <memory>
#include <vector>

#include "gsm_common.h"

namespace gsm {

struct LevelBufs {
    DevBuf<int32_t> rows;  // frontier of this width (input rows of process(width)), plain layout
    DevBuf<int2> pv;       // the same frontier in the compressed layout: (parent row, vertex)
    int64_t cap_rows = 0;  // row capacity reserved for this frontier (per match)
    DevBuf<int64_t> rbeg, rlen, P, tile_ra, cbeg;
    DevBuf<int32_t> clen;
    DevBuf<uint8_t> rpiv, scan_tmp;
    DevBuf<unsigned long long> out_count;
    unsigned long long* stats = nullptr;  // 5 counters for this width's expand launches (per match)
    double rows_in = 0;                   // rows staged by this width's expand launches (per match)
};

struct Workspace {
    std::vector<std::unique_ptr<LevelBufs>> lv;  // index = frontier width 1..k
    DevBuf<uint8_t> cmask;
    DevBuf<unsigned long long> counts, final_count, stats, ovf_n, sched;
    DevBuf<int64_t> ovf_idx;
    DevBuf<uint8_t> la_c1, la_c2, la_ok1;  // k-look-ahead tables (gsm_match_opts.lookahead)
    DevBuf<int32_t> ovf_rows;
    // clique path (gsm_clique.cu): root keys / order, sort temp, global slab, handed-back roots
    DevBuf<int32_t> ck_keys, ck_vals, ck_keys2, ck_vals2, ck_slab, ck_over;
    DevBuf<uint8_t> ck_tmp;
    DevBuf<unsigned long long> ck_bucket, ck_sched;
    DevBuf<int> ck_dmax;
    // pinned host staging for the end-of-match read-back (several D2H copies, one sync)
    unsigned long long* pin = nullptr;
    static constexpr size_t kPin = 1 + kMaxK + 5 * (kMaxK + 1);
    unsigned long long* pinned() {
        if (!pin && cudaMallocHost(&pin, sizeof(unsigned long long) * kPin) != cudaSuccess) {
            (void)cudaGetLastError();
            pin = nullptr;
        }
        return pin;
    }
    Workspace() : lv(kMaxK + 1) {
        for (auto& p : lv) p.reset(new LevelBufs());
    }
    ~Workspace() {
        if (pin) cudaFreeHost(pin);
    }
};

}  // namespace gsm
