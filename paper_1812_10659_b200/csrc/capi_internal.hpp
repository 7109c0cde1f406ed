// Shared pieces of the extern "C" layer: the opaque context type and the
// exception -> status translation (codes as in include/lola_b200.h).
#pragma once

#include <new>
#include <stdexcept>
#include <string>

#include "context.hpp"
#include "lola_eval.hpp"

struct lb_context {
    lb::Context cx;
    explicit lb_context(const lb::Params& p) : cx(p) {}
};

namespace lb::capi {

std::string& last_error();

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const lola::depth_error& e) {
        last_error() = e.what();
        return 4;
    } catch (const lola::magnitude_error& e) {
        last_error() = e.what();
        return 4;
    } catch (const std::invalid_argument& e) {
        last_error() = e.what();
        return 3;
    } catch (const std::out_of_range& e) {
        last_error() = e.what();
        return 3;
    } catch (const std::logic_error& e) {
        last_error() = e.what();
        return 5;
    } catch (const std::bad_alloc&) {
        last_error() = "out of memory";
        return 1;
    } catch (const std::exception& e) {
        last_error() = e.what();
        return 1;
    }
}

inline void need(bool ok, const char* what) {
    if (!ok) throw std::invalid_argument(what);
}

}  // namespace lb::capi
