/* librecd_host: host-side (CPU) helpers of the KJT host -> device path.
 *
 * Row-delta coding of a batch's KJT rows (csrc/host/recd_rowcode.cpp): the
 * H2D copy of the full int64 KJT is what bounds the end-to-end step, and in
 * session-clustered batches (datagen.py:210-250) a history row is usually its
 * predecessor repeated or shifted by one.  Per feature and row, one code:
 *   RECD_ROW_KEY     all L IDs follow in the literals
 *   RECD_ROW_REPEAT  the row equals the previous row (no literal)
 *   RECD_ROW_SHIFT   the row equals previous[1:] + [x] (literal x)
 * librecd's recd_rowcode_decode rebuilds the values on the device (exact).
 * This replaces no reference function: the reference copies the KJT
 * (trainer_sim.py:449-481 consumes host arrays); it is the wire format of the
 * H2D stage (reader.py:160-175). */
#ifndef RECD_HOST_H
#define RECD_HOST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { RECD_ROW_KEY = 0, RECD_ROW_REPEAT = 1, RECD_ROW_SHIFT = 2 };

/* values[f] int64[num_values[f]], offsets[f] int64[batch_size] (row starts,
 * offsets[f][0] == 0); codes_out[f] uint8[batch_size]; lits_out[f]
 * int64[lit_caps[f]]; lit_counts_out[f] = literals written.  num_threads <= 0:
 * all hardware threads.  Returns 0, 1 (bad argument) or 2 (literal capacity
 * exceeded). */
int recd_rowcode_encode(int32_t num_features, int64_t batch_size,
                        const int64_t* const* values, const int64_t* const* offsets,
                        const int64_t* num_values, uint8_t* const* codes_out,
                        int64_t* const* lits_out, const int64_t* lit_caps,
                        int64_t* lit_counts_out, int32_t num_threads);

#ifdef __cplusplus
}
#endif

#endif
