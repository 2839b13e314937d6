// grid.h -- the level/pass geometry lives in the public include tree (it also backs
// ipcomp::LevelTraversal in include/ipcomp/grid.hpp); the kernels' launchers use it from here.
#pragma once
#include "../../include/ipcomp_b200_grid.h"
