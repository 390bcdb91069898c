// dnd/dnd.hpp -- the whole B200 drop-in API (proj/include/dnd/*.hpp names).
#pragma once

#include "dnd/chunking.hpp"
#include "dnd/cluster.hpp"
#include "dnd/dataio.hpp"
#include "dnd/errors.hpp"
#include "dnd/moments.hpp"
#include "dnd/ndarray.hpp"
#include "dnd/pairwise.hpp"
#include "dnd/regression.hpp"
#include "dnd/tile.hpp"
#include "dnd/transport.hpp"
