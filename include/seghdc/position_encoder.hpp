// Forwarding header: the reference's seghdc/position_encoder.hpp API lives in seghdc/seghdc.hpp.
#pragma once
#include "seghdc/seghdc.hpp"
