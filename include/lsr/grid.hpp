// Forwarding header: the reference include path `lsr/grid.hpp` resolves to the
// B200 API, which declares everything the reference header declares
// (see lsr_b200.hpp for the file:line map and which definitions the GPU
// library provides).
#pragma once
#include "lsr/lsr_b200.hpp"
