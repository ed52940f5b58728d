// Drop-in path: the reference includes "radialplan/grid.hpp"; the B200
// facade declares the whole operator API in one header.
#pragma once
#include "../radialplan_b200.hpp"
