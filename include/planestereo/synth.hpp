// synth.hpp — drop-in name for the reference header proj/include/planestereo/synth.hpp;
// of it this build provides wtaOracle (GPU), declared in planestereo.hpp.
#pragma once
#include "planestereo/planestereo.hpp"
