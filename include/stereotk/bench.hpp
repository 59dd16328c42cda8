// Forwarding header: the stereotk:: API of the reference header of the same
// name is declared in stereotk_b200.hpp (GPU-backed drop-in).
#pragma once
#include "stereotk/stereotk_b200.hpp"
