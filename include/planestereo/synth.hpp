// synth.hpp — drop-in name for the reference header proj/include/planestereo/synth.hpp
// (PlanarScene, renderScene, wtaOracle; all on the GPU), declared in planestereo.hpp.
#pragma once
#include "planestereo/planestereo.hpp"
