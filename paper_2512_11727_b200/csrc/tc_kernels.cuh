// Tensor-core (tcgen05, kind::tf32) contractions of the learned backend.
#pragma once
#include <stddef.h>
#include <stdint.h>

struct ecco_ctx;

// A 128-row tile of the fwd contraction: rows [row0, row0 + nrows) all use
// the model in `slot`; `job` indexes the step gate.
struct TcTile {
  int slot;
  int row0;
  int nrows;
  int job;
};

namespace tc {
// Z[r, :] = X[r, :] . W1(slot) + b1 for every tile row.  live_rows: rows
// actually computed (for the algorithmic flop count of the profiler).
void fwd_hidden(ecco_ctx* ctx, const uint16_t* xbase, const int64_t* row_off, const TcTile* tiles,
                int n_tiles, const int* steps, int step, const float* wbase, size_t wstride,
                float* Z, double live_rows);
// Same contraction for training tiles of exactly 128 rows with kind::f16:
// X (bf16, exact) . bf16 W1^T shadow (w1t, [slot][H][F], kept in step with
// the fp32 masters by dw1_update), fp32 accumulation.
void fwd_hidden_bf16(ecco_ctx* ctx, const uint16_t* xbase, const int64_t* row_off,
                     const TcTile* tiles, int n_tiles, const int* steps, int step,
                     const uint16_t* w1t, size_t n_slots, const float* wbase, size_t wstride,
                     float* Z, double live_rows);
// W1(slot[j]) -= lr * X_j^T . dH_j for every job j with step < steps[j]; with
// w1t non-null the bf16 W1^T shadow rows are rewritten too.
void dw1_update(ecco_ctx* ctx, const uint16_t* xbase, const int64_t* row_off, const int* slots,
                const int* steps, int step, int n_jobs, float* wbase, size_t wstride,
                const float* DH, int live_jobs, uint16_t* w1t = nullptr);
}  // namespace tc
