// psg_dense.cuh — the dense cell-pair engine for grids whose
// cells hold many points (clustered data, e.g. BASELINE config 5).
#pragma once

#include <memory>

#include "psg_grid.cuh"
#include "psg_scan.cuh"

namespace psg {

// Buffers reused across solves on one point set.
struct DenseWork {
  DevBuf<float> Xs;                // n x d rows in grid-sorted order
  DevBuf<float> cbox;              // cells x 2nk: per-cell key boxes (lo, hi); only non-empty cells are written
  DevBuf<uint32_t> clist;          // the non-empty cells (any order)
  DevBuf<uint32_t> pa, pb, ptiles, pprefix, stmp;  // surviving cell pairs, tiles per pair, prefix
  DevBuf<uint32_t> hist, gstart, gstrips, gprefix, gtmp;  // Gram path: pairs sorted by A, groups, strip prefix
  DevBuf<unsigned long long> ctr;  // [0] pair count, [1] tile / group cursor, [2] estimate, [3] groups
  uint32_t pair_cap = 0;
};

// Candidate pairs the sparse scan would visit over this grid (zone ignored):
// sum over cells of the stencil sizes.  Synchronises.
uint64_t grid_pair_estimate(const GridIndex& gi, uint64_t cells, cudaStream_t s);

// Every forward-stencil cell pair (A, B) whose key boxes can hold a pair with
// lower bound <= the current threshold is evaluated exhaustively in 128x128
// tiles of canonical FP32 distances (the brute-force kernel's order), from
// grid-sorted rows; pairs inside the band go to the candidate list exactly as
// in the sparse scan.  Tiles are split round-robin over `nparts` parts.
// Returns the number of cell pairs kept.  Synchronises.
uint64_t dense_scan(const ScanArgs& a, const GridIndex& gi, uint64_t cells, const Rows& X, uint32_t n, int d,
                    int nk, Thresholds* th, DenseWork& w, uint32_t part, uint32_t nparts, cudaStream_t s);

}  // namespace psg
