// sched.cuh -- work list of the split-K decode kernels, built on the device from
// lens[] (so a decode iteration needs no host sync and is graph-capturable).
//
// Work items are (slot b, head h, chunk c) with chunks of CHUNK keys counted
// from the slot's live start.  They are handed out DYNAMICALLY (one global
// atomic counter per launch) in longest-first order:
//   phase A: every full 256-key chunk of every slot (all equally long);
//   phase B: the ragged tail chunk of each slot, tails sorted by length,
//            longest first (counting sort over 1..255 in shared memory).
// Greedy longest-first assignment keeps the slowest CTA within a few % of the
// mean on the configs' length mixes (static round-robin was 1.2-1.3x).
// Which CTA runs an item never changes a result: chunk partials are merged in
// chunk order (batch invariance).
#pragma once
#include "common.cuh"
#include "kernels.h"

namespace baton {

struct WorkSched {
    int32_t prefixA[MAX_SLOTS + 1];   // exclusive prefix of full-chunk items per slot
    int32_t tails[MAX_SLOTS];         // slots with a ragged tail, longest tail first
    int32_t bins[CHUNK];
    int32_t lens[MAX_SLOTS];
    int32_t pad[MAX_SLOTS];
    int32_t totalA, ntails;
};

// Warp-collective (all 32 lanes of one warp).  H = heads per slot in the item space.
BATON_DEV void sched_build(WorkSched &ws, const int32_t *lens, const int32_t *pad, int B, int H,
                           int lane) {
    for (int i = lane; i < CHUNK; i += 32) ws.bins[i] = 0;
    int running = 0;
    for (int b0 = 0; b0 < B; b0 += 32) {
        const int b = b0 + lane;
        int L = 0;
        if (b < B) {
            L = lens[b];
            ws.lens[b] = L;
            ws.pad[b] = pad[b];
        }
        const int n = (L > 0 ? L / CHUNK : 0) * H;
        int incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(FULL_MASK, incl, o);
            if (lane >= o) incl += t;
        }
        if (b < B) ws.prefixA[b] = running + incl - n;
        running += __shfl_sync(FULL_MASK, incl, 31);
    }
    if (lane == 0) ws.prefixA[B] = running;
    if (lane == 0) ws.totalA = running;
    __syncwarp();
    // counting sort of tails (length L % CHUNK in 1..255) by length, descending
    for (int b = lane; b < B; b += 32) {
        const int r = ws.lens[b] > 0 ? ws.lens[b] % CHUNK : 0;
        if (r) atomicAdd(&ws.bins[r], 1);
    }
    __syncwarp();
    // lane owns bins (descending) CHUNK-1-8*lane-i, i < 8; exclusive scan -> start offsets
    int cnt[8];
    int local = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int r = CHUNK - 1 - (lane * 8 + i);
        cnt[i] = ws.bins[r];
        local += cnt[i];
    }
    int incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(FULL_MASK, incl, o);
        if (lane >= o) incl += t;
    }
    int start = incl - local;
    const int ntails = __shfl_sync(FULL_MASK, incl, 31);
    __syncwarp();
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const int r = CHUNK - 1 - (lane * 8 + i);
        ws.bins[r] = start;     // becomes a placement cursor
        start += cnt[i];
    }
    __syncwarp();
    for (int b = lane; b < B; b += 32) {
        const int r = ws.lens[b] > 0 ? ws.lens[b] % CHUNK : 0;
        if (r) ws.tails[atomicAdd(&ws.bins[r], 1)] = b;
    }
    if (lane == 0) ws.ntails = ntails;
    __syncwarp();
}

BATON_DEV int sched_total(const WorkSched &ws, int H) { return ws.totalA + ws.ntails * H; }

// Decode item w; `b` is a forward-scan cursor for phase A (w increases per caller).
BATON_DEV void sched_item(const WorkSched &ws, int w, int H, int &b, int &c, int &h) {
    if (w < ws.totalA) {
        while (ws.prefixA[b + 1] <= w) ++b;
        const int rem = w - ws.prefixA[b];
        c = rem / H;
        h = rem - c * H;
    } else {
        const int j = w - ws.totalA;
        const int k = j / H;
        h = j - k * H;
        const int bt = ws.tails[k];
        c = ws.lens[bt] / CHUNK;
        b = bt;
    }
}

// Dynamic work counter: counters[0] = next item, counters[1] = CTAs done.  The
// last CTA to finish resets both for the next (stream-ordered) launch.
BATON_DEV int sched_next(int32_t *counters) { return atomicAdd(&counters[0], 1); }
BATON_DEV void sched_done(int32_t *counters) {
    __threadfence();
    if (atomicAdd(&counters[1], 1) == (int)gridDim.x - 1) {
        atomicExch(&counters[0], 0);
        atomicExch(&counters[1], 0);
    }
}

}  // namespace baton
