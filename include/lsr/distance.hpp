// Forwarding header: the reference include path `lsr/distance.hpp` resolves to the
// B200 host API (see lsr_b200.hpp for the reference file:line map).
#pragma once
#include "lsr/lsr_b200.hpp"
