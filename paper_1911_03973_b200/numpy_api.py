"""NumPy in, NumPy out: the device package behind the reference's exact call surface.

The reference package ``ebsolve`` (/root/reference/pkg/src/ebsolve/__init__.py:53-92) takes
and returns host NumPy arrays (read-only on its frozen data classes, mesh.py:53-54,90-91,
operators.py:46-47) and SciPy sparse matrices (reference.py:25-39).  The device package
returns CUDA tensors.  This module closes that last gap for a caller that switches over
without touching its code: every entry point of a device module is re-exposed so that

  * arguments pass through unchanged (the device entry points accept NumPy arrays), with
    facade objects replaced by the device objects they hold and user callbacks handed
    NumPy copies of the tensors the solver passes them (solvers.py:137-149);
  * results come back as host arrays: float64 / int64 ndarrays for tensors (the int32
    device connectivity widens to the reference's int64), ``scipy.sparse.csr_matrix`` for
    sparse CSR tensors, and facade objects for the data classes that hold tensors (``Mesh``,
    ``IndexArrays``, ``ElementBatch``, ``DirichletData``, the experiment report), whose
    array attributes are converted once, cached and read-only like the reference's.

Nothing is computed here: every call lands in the device package (libebs.so); the module
only moves results across PCIe, so it is the convenience boundary, not the fast one (device
tensors stay resident through ``paper_1911_03973_b200`` itself).  ``compat/ebsolve`` is an
import-name shim over this module: with ``paper_1911_03973_b200/compat`` on ``sys.path``,
``import ebsolve`` (and ``ebsolve.cli``, ``.mesh``, ``.elements``, ``.operators``,
``.solvers``, ``.spectrum``, ``.reference``, ``python -m ebsolve.cli``) resolve here, which
is how the reference's own test-suite is run against the CUDA path
(``scripts/run_reference_tests.py``).
"""

from __future__ import annotations

import dataclasses
import functools
import importlib
import inspect
import sys
import types

import numpy as np
import torch

_PKG = __name__.rsplit(".", 1)[0]

# device class -> facade class (filled by _facade_class)
_FACADES: dict[type, type] = {}
# device module name -> facade module
_MODULES: dict[str, types.ModuleType] = {}


def _host_array(t: torch.Tensor, frozen: bool) -> np.ndarray:
    a = t.detach().to("cpu").numpy()
    if a.dtype == np.int32:
        a = a.astype(np.int64)
    elif not a.flags.owndata and t.device.type == "cpu":
        a = a.copy()
    if frozen:
        a.setflags(write=False)
    return a


def _host_sparse(t: torch.Tensor):
    import scipy.sparse as sp
    t = t.to("cpu")
    if t.layout != torch.sparse_csr:
        t = t.to_sparse_csr()
    return sp.csr_matrix((t.values().numpy().copy(), t.col_indices().numpy().copy(),
                          t.crow_indices().numpy().copy()), shape=tuple(t.shape))


def to_host(v, frozen: bool = False):
    """Device result -> what the reference would have returned."""
    if isinstance(v, torch.Tensor):
        if v.layout != torch.strided:
            return _host_sparse(v)
        return _host_array(v, frozen)
    cls = type(v)
    if cls in _FACADES:
        return _FACADES[cls]._adopt(v)
    if isinstance(v, tuple) and not hasattr(v, "_fields"):
        return tuple(to_host(e, frozen) for e in v)
    if isinstance(v, list):
        return [to_host(e, frozen) for e in v]
    if isinstance(v, dict):
        return {k: to_host(e, frozen) for k, e in v.items()}
    if _holds_tensors(v):
        return _facade_class(cls)._adopt(v)
    return v


def _holds_tensors(v) -> bool:
    """A data class instance of the device package with a tensor (or a data class that
    holds one) among its fields."""
    if not dataclasses.is_dataclass(v) or isinstance(v, type):
        return False
    if not type(v).__module__.startswith(_PKG):
        return False
    for f in dataclasses.fields(v):
        e = getattr(v, f.name, None)
        if isinstance(e, torch.Tensor) or type(e) in _FACADES or _holds_tensors(e):
            return True
        if isinstance(e, dict) and any(_holds_tensors(x) or type(x) in _FACADES
                                       for x in e.values()):
            return True
    return False


def to_device_arg(v):
    """Facade objects -> the device objects they hold; callables -> callables whose
    arguments are converted to host arrays (solver callbacks, source functions take NumPy
    coordinates already)."""
    if isinstance(v, _Facade):
        return v._obj
    if isinstance(v, tuple) and not hasattr(v, "_fields"):
        return tuple(to_device_arg(e) for e in v)
    if isinstance(v, list):
        return [to_device_arg(e) for e in v]
    if isinstance(v, dict):
        return {k: to_device_arg(e) for k, e in v.items()}
    dev = getattr(v, "__device_function__", None)
    if dev is not None:
        return dev
    if isinstance(v, (types.FunctionType, types.MethodType, functools.partial)):
        return _host_callback(v)
    return v


def _host_callback(fn):
    @functools.wraps(fn)
    def call(*args, **kwargs):
        out = fn(*[to_host(a) for a in args], **{k: to_host(a) for k, a in kwargs.items()})
        return to_device_arg(out)
    return call


def _host_function(fn):
    """A device-package function with the reference's host-array calling convention."""
    @functools.wraps(fn)
    def call(*args, **kwargs):
        return to_host(fn(*to_device_arg(args), **to_device_arg(kwargs)))
    call.__device_function__ = fn
    return call


class _Facade:
    """Host view of one device object: attributes converted on first read and cached
    (arrays read-only, like the reference's frozen data classes); methods take and return
    host arrays."""

    _device_class: type = object
    __slots__ = ("_obj", "_cache")

    def __init__(self, *args, **kwargs):
        obj = type(self)._device_class(*to_device_arg(args), **to_device_arg(kwargs))
        object.__setattr__(self, "_obj", obj)
        object.__setattr__(self, "_cache", {})

    @classmethod
    def _adopt(cls, obj):
        self = object.__new__(cls)
        object.__setattr__(self, "_obj", obj)
        object.__setattr__(self, "_cache", {})
        return self

    def __getattr__(self, name):
        if name.startswith("__") and name.endswith("__"):
            raise AttributeError(name)
        cache = object.__getattribute__(self, "_cache")
        if name in cache:
            return cache[name]
        obj = object.__getattribute__(self, "_obj")
        v = getattr(obj, name)
        if inspect.ismethod(v) or inspect.isfunction(v):
            w = _host_function(v)
        else:
            w = to_host(v, frozen=True)
        frozen = getattr(type(obj), "__dataclass_params__", None)
        if frozen is None or frozen.frozen or isinstance(v, torch.Tensor):
            cache[name] = w
        return w

    def __setattr__(self, name, value):
        obj = object.__getattribute__(self, "_obj")
        params = getattr(type(obj), "__dataclass_params__", None)
        if params is None or params.frozen:
            raise dataclasses.FrozenInstanceError(f"cannot assign to field {name!r}")
        setattr(obj, name, to_device_arg(value))
        object.__getattribute__(self, "_cache").pop(name, None)

    def __eq__(self, other):
        if isinstance(other, _Facade):
            other = other._obj
        return self._obj == other

    def __hash__(self):
        return hash(self._obj)

    def __repr__(self):
        return repr(self._obj)


def _facade_class(dev_cls: type) -> type:
    cls = _FACADES.get(dev_cls)
    if cls is None:
        cls = type(dev_cls.__name__, (_Facade,), {
            "_device_class": dev_cls, "__slots__": (), "__doc__": dev_cls.__doc__,
            "__module__": __name__, "__qualname__": dev_cls.__name__})
        _FACADES[dev_cls] = cls
    return cls


# the device data classes whose fields hold tensors (directly or through one another): seen
# through the facade they are facade classes, so constructing one from host arrays and reading
# its fields both follow the reference's convention
_TENSOR_CLASSES = frozenset({"Mesh", "IndexArrays", "ElementBatch", "DirichletData", "SolverRun",
                             "ExperimentReport"})


def _tensor_dataclass(cls) -> bool:
    return (isinstance(cls, type) and dataclasses.is_dataclass(cls)
            and cls.__module__.startswith(_PKG) and cls.__name__ in _TENSOR_CLASSES)


class _FacadeModule(types.ModuleType):
    """A device module seen through the host-array convention.  Functions are wrapped on
    first access; data classes with tensor fields become facade classes; everything else
    (constants, pure host data classes) is the device module's own object.  Assignments
    (monkeypatched constants and functions, test_reference.py:106, test_cli.py:194) land
    in the device module, so the code that runs sees them."""

    def __init__(self, dev: types.ModuleType, name: str):
        super().__init__(name, dev.__doc__)
        self.__dict__["__device_module__"] = dev
        self.__dict__["__wrapped_names__"] = {}
        if hasattr(dev, "__all__"):
            self.__dict__["__all__"] = list(dev.__all__)

    def __getattr__(self, name):
        if name.startswith("__") and name.endswith("__"):
            raise AttributeError(name)
        dev = self.__dict__["__device_module__"]
        v = getattr(dev, name)
        cached = self.__dict__["__wrapped_names__"].get(name)
        if cached is not None and cached[0] is v:
            return cached[1]
        if isinstance(v, types.ModuleType):
            w = facade(v) if v.__name__.startswith(_PKG) else v
        elif isinstance(v, type):
            w = _facade_class(v) if (v in _FACADES or _tensor_dataclass(v)) else v
        elif inspect.isfunction(v) and getattr(v, "__device_function__", None) is None \
                and (v.__module__ or "").startswith(_PKG):
            w = _host_function(v)
        else:
            w = v
        self.__dict__["__wrapped_names__"][name] = (v, w)
        return w

    def __setattr__(self, name, value):
        if name.startswith("__") and name.endswith("__"):
            self.__dict__[name] = value
            return
        if isinstance(value, types.ModuleType):  # the import system binding a submodule
            self.__dict__[name] = value
            return
        dev = self.__dict__["__device_module__"]
        inner = getattr(value, "__device_function__", None)
        if inner is not None:
            value = inner
        elif isinstance(value, type) and issubclass(value, _Facade):
            value = value._device_class
        elif inspect.isfunction(value) or inspect.ismethod(value):
            # a host-convention replacement for a device function (monkeypatch): the device
            # code calls it with device objects and uses what it returns
            value = _host_callback(value)
        setattr(dev, name, value)

    def __delattr__(self, name):
        delattr(self.__dict__["__device_module__"], name)

    def __dir__(self):
        return sorted(set(dir(self.__dict__["__device_module__"])))


def facade(dev) -> types.ModuleType:
    """The host-array view of a device module (by module object or by name relative to the
    package, e.g. ``facade("cli")``)."""
    if isinstance(dev, str):
        dev = importlib.import_module(f"{_PKG}.{dev}" if dev else _PKG)
    mod = _MODULES.get(dev.__name__)
    if mod is None:
        mod = _FacadeModule(dev, dev.__name__ + "[numpy]")
        _MODULES[dev.__name__] = mod
    return mod


_SUBMODULES = ("cli", "mesh", "elements", "operators", "solvers", "spectrum", "reference",
               "sparse")


def install(alias: str = "ebsolve", package_dir: str | None = None) -> types.ModuleType:
    """Register the facade in ``sys.modules`` under the reference's import name: ``alias`` for
    the package and ``alias.<module>`` for its modules.

    With ``package_dir`` (the ``compat/ebsolve`` shim) the package facade gets that directory
    as its ``__path__`` and ``alias.cli`` is left to the shim's ``cli.py`` file, so that
    ``python -m ebsolve.cli`` (test_cli.py:218-225) has a module spec to run."""
    root = facade("")
    sys.modules[alias] = root
    if package_dir is not None:
        root.__dict__["__path__"] = [package_dir]
        root.__dict__["__package__"] = alias
    for sub in _SUBMODULES:
        root.__dict__[sub] = facade(sub)
        if package_dir is None or sub != "cli":
            sys.modules[f"{alias}.{sub}"] = facade(sub)
    return root


def __getattr__(name):
    """``from paper_1911_03973_b200.numpy_api import residual`` etc.: the package's
    exports in the host-array convention."""
    if name.startswith("__"):
        raise AttributeError(name)
    return getattr(facade(""), name)
