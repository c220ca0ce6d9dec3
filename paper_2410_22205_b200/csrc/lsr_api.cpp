// lsr_api.cpp — the C++ `lsr::` face (include/lsr/lsr_b200.hpp) over the C
// ABI. Error behaviour follows the reference: checks that the reference
// performs before touching data (evolve.cpp:42-46) throw before any device
// work; a non-finite update throws NumericalError after `out` is written.
#include <string>

#include "lsr/lsr_b200.hpp"

namespace lsr {

void throw_status(int status) {
    if (status == LSR_OK) return;
    const std::string msg = lsr_cuda_last_error_string();
    switch (status) {
        case LSR_ERR_CONFIG: throw ConfigError(msg);
        case LSR_ERR_NUMERICAL: throw NumericalError(msg);
        case LSR_ERR_OUT_OF_DOMAIN: throw OutOfDomainError(msg);
        case LSR_ERR_NO_INTERFACE: throw NoInterfaceError(msg);
        case LSR_ERR_CUDA: throw CudaError(msg);
        default: throw Error(msg);
    }
}

void sl_step(const ScalarField& phi, const DistanceField& dist, const BandMask& mask, const StepConfig& cfg,
             double energy_p, ScalarField& out) {
    cfg.validate();
    if (!(phi.grid == dist.field.grid) || !(phi.grid == mask.grid))
        throw ConfigError("sl_step: phi, dist and mask must share one grid");
    if (cfg.p > 1 && !(energy_p > 0.0)) throw Error("sl_step: energy must be positive for p > 1");
    const Grid& g = phi.grid;
    if (!(out.grid == g) || out.values.size() != phi.values.size()) out = ScalarField(g);
    const lsr_grid cg = g.c();
    const lsr_step_cfg cc = cfg.c();
    std::int64_t bad = -1;
    throw_status(lsr_cuda_sl_step_host(&cg, phi.values.data(), dist.field.values.data(), mask.active.data(),
                                       static_cast<std::int64_t>(mask.active.size()), &cc, energy_p,
                                       out.values.data(), &bad));
}

}  // namespace lsr
