// Fused pass entry (qs_apply_fused).  Validation + per-op dispatch; the
// tile kernel lives below once written.
#include <string>

#include "common.cuh"
#include "internal.h"

namespace qsb {

int run_fused(qs_state *s, const int32_t *tile_qubits, int ntile, const qs_op *ops, int nops) {
    const int n = s->num_qubits;
    uint64_t tile_mask = 0;
    for (int i = 0; i < ntile; ++i) {
        if (tile_qubits[i] < 0 || tile_qubits[i] >= n)
            return set_error(QS_ERR_INDEX, "tile qubit " + std::to_string(tile_qubits[i]) +
                                               " out of range");
        tile_mask |= 1ull << tile_qubits[i];
    }
    for (int i = 0; i < nops; ++i) {
        const qs_op &op = ops[i];
        if (op.target < 0 || op.target >= n)
            return set_error(QS_ERR_INDEX, "op target out of range");
        if (op.ctrl_mask >> n) return set_error(QS_ERR_INDEX, "op control out of range");
        if ((op.ctrl_mask >> op.target) & 1ull)
            return set_error(QS_ERR_VALUE, "control and target must differ");
        if (op.kind == QS_OP_PAIR && !((tile_mask >> op.target) & 1ull))
            return set_error(QS_ERR_VALUE, "pair-op target " + std::to_string(op.target) +
                                               " is not a tile qubit");
        if (op.kind != QS_OP_PAIR && op.kind != QS_OP_PHASE)
            return set_error(QS_ERR_VALUE, "unknown op kind");
    }
    for (int i = 0; i < nops; ++i) {
        const qs_op &op = ops[i];
        int rc = op.kind == QS_OP_PHASE
                     ? launch_phase(s, op.ctrl_mask | (1ull << op.target), make_float2(op.m[6], op.m[7]))
                     : launch_sweep(s, op.target, op.ctrl_mask, op.m);
        if (rc) return rc;
    }
    return QS_OK;
}

}  // namespace qsb
