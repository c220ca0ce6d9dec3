// Forwarding header: the reference include path `lsr/reinit.hpp` resolves to the
// B200 API, which declares everything the reference header declares
// (see lsr_b200.hpp for the file:line map and which definitions the GPU
// library provides).
#pragma once
#include "lsr/lsr_b200.hpp"
