// Forwarding header: the reference's seghdc/pixel_pipeline.hpp API lives in seghdc/seghdc.hpp.
#pragma once
#include "seghdc/seghdc.hpp"
