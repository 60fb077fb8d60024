// Forwarding header: the reference's seghdc/errors.hpp API lives in seghdc/seghdc.hpp.
#pragma once
#include "seghdc/seghdc.hpp"
